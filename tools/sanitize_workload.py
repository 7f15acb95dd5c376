"""Workload for tools/sanitize.sh: stencil (2 instances, n = 70000) and the
classified tree reduction (300 instances, n = 1024) through the C ABI."""
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
