"""Workload for tools/sanitize.sh: stencil (2 instances, n = 70000) and the
round-2 paths at the end (oversized bucket, prepass, LSD sort, work-groups),
classified tree reduction (300 instances, n = 1024) through the C ABI, and
the interleaving explorer on K_inc (n = 4, both scheduling modes)."""
import sys, os; sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1308_3203_b200 import rc_load_program, rc_run
from workloads import kernels as K, inputs as I
p = K.program(K.STENCIL); prog = rc_load_program(p.bytecode)
ins = I.cfg5_inputs(0, 2, 70000)
r = rc_run(prog, 70000, [torch.from_numpy(x).cuda() for x in ins])
print("stencil ok", r.stats["checked_accesses"])
p = K.program(K.TREE_OFF_BY_ONE); prog = rc_load_program(p.bytecode)
ins = I.cfg3_inputs(0, 300, 1024)
r = rc_run(prog, 1024, [torch.from_numpy(x).cuda() for x in ins], classify_rw=True)
print("tree ok", len(r.reports))
from oracle import oracle as orc  # noqa: E402  (test infrastructure: the explorer's start state)
from paper_1308_3203_b200 import rc_explore  # noqa: E402
p = K.program(K.BENIGN["K_inc"]); prog = rc_load_program(p.bytecode)
_, heap, regs, pc, st = orc.state_at(p.bytecode, 4, [np.array([40], np.int32), np.zeros(4, np.int32)], 0)
args = dict(regs=torch.from_numpy(regs).cuda(), pc=torch.from_numpy(pc.astype(np.int32)).cuda(),
            status=torch.from_numpy(st).cuda(), sizes=[1, 4], index_end=1 << 12, cap=64, max_len=16)
for red in (True, False):
    r = rc_explore(prog, 4, torch.from_numpy(heap.astype(np.int32)).cuda(), reduced=red, **args)
    print("explore ok", r.n_schedules, r.n_differ)
# round 2 paths: an oversized bucket (global counting sort), the prepass
# direct-commit mode, the onesweep LSD path, work-groups
p = K.program(K.BENIGN["K_inc"]); prog = rc_load_program(p.bytecode)
ins = I.cfg2_inputs(0, 2, 20000)
r = rc_run(prog, 20000, [torch.from_numpy(x).cuda() for x in ins])
print("oversized bucket ok", len(r.reports))
p = K.program(K.STENCIL); prog = rc_load_program(p.bytecode)
ins = I.cfg5_inputs(0, 2, 70000)
r = rc_run(prog, 70000, [torch.from_numpy(x).cuda() for x in ins], prepass=True)
print("prepass ok", r.stats["checked_accesses"])
os.environ["RC_SORT_LSD"] = "1"
p = K.program(K.TREE_OFF_BY_ONE); prog = rc_load_program(p.bytecode)
ins = I.cfg3_inputs(0, 40, 1024)
r = rc_run(prog, 1024, [torch.from_numpy(x).cuda() for x in ins])
print("lsd ok", len(r.reports))
del os.environ["RC_SORT_LSD"]
r = rc_run(prog, 512, [torch.from_numpy(x).cuda() for x in ins], n_groups=2)
print("groups ok", len(r.reports))
# K1c (the interval kernel compiled per program): bucket writes + fresh start
# + report snapshot (stencil), reports / fuel (tree), the plane variant after
# a bucket overflow, direct mode, and the hand-back to K1 (rc_k1c_fix)
os.environ["RC_JIT"] = "1"
p = K.program(K.STENCIL); prog = rc_load_program(p.bytecode)
ins = I.cfg5_inputs(0, 2, 70000)
r = rc_run(prog, 70000, [torch.from_numpy(x).cuda() for x in ins])
r = rc_run(prog, 70000, [torch.from_numpy(x).cuda() for x in ins], prepass=True)
print("k1c stencil ok", r.stats["checked_accesses"], prog.jit_kernels())
p = K.program(K.TREE_OFF_BY_ONE); prog = rc_load_program(p.bytecode)
ins = I.cfg3_inputs(0, 40, 1024)
r = rc_run(prog, 1024, [torch.from_numpy(x).cuda() for x in ins])
print("k1c tree ok", len(r.reports), prog.jit_kernels())
p = K.program(K.BENIGN["K_inc"]); prog = rc_load_program(p.bytecode)
ins = I.cfg2_inputs(0, 2, 20000)
r = rc_run(prog, 20000, [torch.from_numpy(x).cuda() for x in ins])
print("k1c oversized bucket ok", len(r.reports), prog.jit_kernels())
from workloads.asm import assemble  # noqa: E402
p = assemble(""".arrays X Y
    tid r0
    const r1, 2
    lt r2, r0, r1
    br r2, left, right
left:
    bar
    const r5, 0
    ld r3, X, r5
    ld r4, X, r0
    ld r6, Y, r0
    exit
right:
    bar
    const r5, 0
    st X, r5, r0
    exit
"""); prog = rc_load_program(p.bytecode)
ins = [np.arange(600, dtype=np.int32).reshape(2, 300), np.zeros((2, 300), np.int32)]
r = rc_run(prog, 300, [torch.from_numpy(x).cuda() for x in ins])
print("k1c hand-back ok", len(r.reports), prog.jit_kernels())
