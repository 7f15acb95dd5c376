"""K1c (jit.cpp) on the GPU: the kernel compiled per program really runs
(tests/test_gpu_parity.py runs every parity case under K1 and under K1c;
here what is specific to K1c): the size threshold, the hand-back to K1 when a
work-item has more records than K1c's planes, and the direct-commit mode."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from workloads import inputs as I  # noqa: E402
from workloads import kernels as K  # noqa: E402
from workloads.asm import assemble  # noqa: E402

from test_gpu_parity import assert_parity  # noqa: E402


@pytest.fixture(scope="module")
def rc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1308_3203_b200 as pkg
    pkg.lib()
    return pkg


def both(rc, p, n, ins, **kw):
    prog = rc.rc_load_program(p.bytecode)
    g = rc.rc_run(prog, n, [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in ins], **kw)
    o = oracle.run(p.bytecode, n, ins, instance_offset=kw.get("instance_offset", 0))
    return prog, g, o


def test_k1c_compiled_and_used(rc, monkeypatch):
    monkeypatch.setenv("RC_JIT", "1")
    p = K.program(K.STENCIL)
    n = 3000
    ins = I.cfg5_inputs(0, 5, n)
    prog, g, o = both(rc, p, n, ins)
    assert_parity(g, o, ins)
    assert prog.jit_kernels() == 1
    # the same shape again: the cached kernel (no second compile)
    g2 = rc.rc_run(prog, n, [torch.from_numpy(x).cuda() for x in ins])
    assert_parity(g2, o, ins)
    assert prog.jit_kernels() == 1


def test_k1c_size_threshold(rc, monkeypatch):
    """Without RC_JIT the kernel is compiled only for batches of >= 2^20
    lanes (RC_JIT_MIN_LANES); RC_JIT=0 never compiles."""
    monkeypatch.delenv("RC_JIT", raising=False)
    p = K.program(K.STENCIL)
    ins = I.cfg5_inputs(1, 2, 1000)
    prog, g, o = both(rc, p, 1000, ins)
    assert prog.jit_kernels() == 0
    assert_parity(g, o, ins)
    monkeypatch.setenv("RC_JIT_MIN_LANES", "1000")
    prog, g, o = both(rc, p, 1000, ins)
    assert prog.jit_kernels() == 1
    assert_parity(g, o, ins)
    monkeypatch.setenv("RC_JIT", "0")
    prog, g, o = both(rc, p, 1000, ins)
    assert prog.jit_kernels() == 0


def test_k1c_bail_to_interpreter(rc, monkeypatch):
    """After a barrier divergence an instance logs every read: the work-items
    after `left` log three reads where K1c's planes hold one record (the
    static bound with the write-set elision), so K1c hands the interval back
    to K1 — same reports, heaps and counters as the oracle."""
    monkeypatch.setenv("RC_JIT", "1")
    src = """
.arrays X Y
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
"""
    p = assemble(src)
    for n in (5, 300):
        ins = [np.arange(2 * n, dtype=np.int32).reshape(2, n), np.zeros((2, n), np.int32)]
        prog, g, o = both(rc, p, n, ins)
        assert_parity(g, o, ins)
        assert prog.jit_kernels() == 1
        assert any(t[4] == 1 for t in o.report_tuples())


def test_k1c_direct_commit(rc, monkeypatch):
    """RC_OPT_PREPASS (the stencil proved conflict-free): K1c commits at the
    end of each work-item's interval, like K1's direct mode."""
    monkeypatch.setenv("RC_JIT", "1")
    p = K.program(K.STENCIL)
    n = 4096
    ins = I.cfg5_inputs(2, 3, n)
    prog, g, o = both(rc, p, n, ins, prepass=True)
    assert_parity(g, o, ins)
    assert prog.jit_kernels() == 1


def test_k1c_random_kernels_many_shapes(rc, monkeypatch):
    """Random tiny kernels (every opcode, branches, loops with fuel) with
    K1c forced: each program is compiled for its shape and matches the
    oracle element by element."""
    monkeypatch.setenv("RC_JIT", "1")
    rng = np.random.default_rng(11)
    used = 0
    for i in range(40):
        p = K.random_tiny_kernel(rng)
        n = int(rng.integers(2, 5))
        ins = [rng.integers(-3, 4, size=(3, n + 2)).astype(np.int32) for _ in range(2)]
        prog = rc.rc_load_program(p.bytecode)
        g = rc.rc_run(prog, n, [torch.from_numpy(x).cuda() for x in ins], fuel_per_interval=64)
        o = oracle.run(p.bytecode, n, ins, fuel=64)
        assert_parity(g, o, ins)
        used += prog.jit_kernels()
    assert used > 20
