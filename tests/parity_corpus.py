"""Opcode-coverage corpus of the GPU parity tests (test infrastructure).

Every entry is (name, Program, n, inputs, rc_run keyword arguments).  Together they execute every
RCB1 opcode of include/rc.h (the §3 grammar lowered):
`tests/test_opcode_coverage.py` checks that on the oracle (CPU), and
`tests/test_gpu_parity.py::test_opcode_corpus` runs each entry through the
C ABI and compares it with the oracle element by element while summing the
oracle's per-opcode execution counts.  No method arithmetic lives here.
"""
from __future__ import annotations

import numpy as np

from workloads import inputs as I
from workloads import kernels as K
from workloads.asm import OPCODES, assemble

# every instruction that makes a work-item stop: ⊥ (DIV0, ASSERT, OOB),
# ⊤ (assume), FUEL (a loop without barrier), divergent barriers, exit
ERROR_KINDS = """
.arrays A
    tid r0
    const r1, 0
    const r2, 1
    eq r3, r0, r1
    br r3, div0, n1
div0:
    div r4, r2, r1
n1:
    eq r3, r0, r2
    lnot r3, r3
    assert r3
    const r5, 2
    eq r3, r0, r5
    lnot r3, r3
    assume r3
    const r5, 3
    eq r3, r0, r5
    br r3, spin, more
spin:
    jmp spin
more:
    const r5, 5
    lt r3, r0, r5
    br r3, b1, b2
b1:
    bar
    st A, r0, r0
    exit
b2:
    bar
    exit
"""

# register-to-register ops on loaded operands, MOV and LNOT included, every
# result stored to a private row of O (no race; a wrong opcode shows in O)
_ALU = ["add", "sub", "mul", "div", "mod", "min", "max", "and", "or", "xor", "lt", "eq", "land", "mov", "lnot"]


def _alu_kernel():
    src = [".arrays X Y O", " tid r0", " ld r1, X, r0", " ld r2, Y, r0", f" const r4, {len(_ALU)}",
           " mul r5, r0, r4"]
    for op in _ALU:
        src += [f" {op} r3, r1" if op in ("mov", "lnot") else f" {op} r3, r1, r2", " st O, r5, r3",
                " addi r5, r5, 1"]
    src += [" exit"]
    return assemble("\n".join(src))


def _alu_inputs():
    rng = np.random.default_rng(3)
    vals = np.concatenate([[0, 1, -1, 2**31 - 1, -2**31, 7, -7], rng.integers(-2**31, 2**31, 40)]).astype(np.int32)
    X = np.repeat(vals, len(vals))[None, :]
    Y = np.tile(vals, len(vals))[None, :].copy()
    Y[Y == 0] = 3
    return [X, Y, np.zeros((1, X.shape[1] * len(_ALU)), np.int32)]


def _tiny(seed, count):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(count):
        n = int(rng.integers(1, 70))
        p = K.random_tiny_kernel(rng, n_arrays=2, n_regs=5, n_commands=int(rng.integers(3, 12)), size=5)
        ins = [rng.integers(-3, 4, size=(int(rng.integers(1, 4)), 5)).astype(np.int32)]
        ins.append(rng.integers(-3, 4, size=(ins[0].shape[0], 5)).astype(np.int32))
        out.append((f"tiny{seed}_{i}", p, n, ins, {}))
    return out


def _cfg4_full(seed, n=300):
    ins = I.cfg4_inputs(0, 4, n)
    ins[3][:, 40:80] += 1  # dense index perturbation: input-dependent WW / RW
    return (f"cfg4_full_isa_{seed}", K.random_stencil_kernel(seed, isa="full"), n, ins, {})


GROUPS = """
.arrays A B
    lid   r0
    gid   r1
    lsize r2
    mul   r3, r1, r2
    add   r3, r3, r0       ; = tid
    st    A, r3, r1        ; A[tid] := gid (disjoint)
    const r4, 0
    st    B, r4, r2        ; B[0] := n in every group (IG_WW_BENIGN)
    exit
"""


def corpus():
    c = [("fig1", K.program(K.FIG1), 8, I.cfg1_inputs()),
         ("fig1_guarded", K.program(K.FIG1_GUARDED), 8, I.cfg1_inputs()),
         ("fig2", K.program(K.FIG2), 2, [np.array([[7, 9, 5]], np.int32), np.array([[42]], np.int32)]),
         ("error_kinds", assemble(ERROR_KINDS), 40, [np.zeros((3, 40), np.int32)]),
         ("tree_off_by_one", K.program(K.TREE_OFF_BY_ONE), 256, I.cfg3_inputs(0, 4, 256)),
         ("stencil", K.program(K.STENCIL), 500, I.cfg5_inputs(0, 2, 500)),
         ("alu", _alu_kernel(), 47 * 47, _alu_inputs()),
         ("many_writes", K.many_writes_kernel(), 40, [np.arange(2 * (64 * 40 + 6), dtype=np.int32).reshape(2, -1),
                                                      np.zeros((2, 40), np.int32)])]
    c = [x + ({},) for x in c]
    c.append(("groups", assemble(GROUPS), 33, [np.zeros((2, 99), np.int32), np.zeros((2, 1), np.int32)],
              {"n_groups": 3}))
    c += [_cfg4_full(s) for s in range(4)]
    c += _tiny(2024, 40)
    return c


FUEL = 300  # per-interval fuel of the corpus runs (ERROR_KINDS spins)


def all_opcodes():
    return sorted(OPCODES.values())
