"""The symbolic NoRace pre-pass (include/rc.h rc_prove; SURVEY.md §8(f) row 4;
PAPER.md:318-447).  Host code only: these tests run without a GPU.

Pins, each derived from the paper and App. A by hand:
  * the 3-point stencil (App. A.5) and the race-free tree reduction (A.4) are
    race-free for every input: NO_CONFLICT;
  * Fig. 1 verbatim reads A[-1] at tid 0 (A.1): OOB; the guarded variant has
    the RW race on R[tid+1] after the barrier: RW;
  * the off-by-one tree reduction reads A[1024] at tid 512 (A.4): OOB;
  * the benign suite (A.3): A[0]:=7, A[0]:=B[0] and the
    last-value kernel write provably equal values (the paper's NoRace holds:
    NORACE); A[0]:=tid and A[0]:=B[tid] may write different values (WW);
    K_inc reads what another work-item writes (RW);
  * Fig. 2: the RW race on A[tid+1] in its second interval.
Soundness against the concrete semantics (the oracle): whenever the prover
claims NO_CONFLICT the oracle reports nothing, and NORACE only WW_BENIGN, on
random inputs of random kernels; and against the paper's all-schedules
definition: every interval of such a kernel has exactly one
reachable end heap (brute-force enumeration, n <= 3).
"""
import numpy as np
import pytest

import oracle
from workloads import inputs as I
from workloads import kernels as K
from workloads.asm import assemble


@pytest.fixture(scope="module")
def rc():
    import paper_1308_3203_b200 as pkg
    pkg.lib()
    return pkg


def prove(rc, src, n, sizes, **kw):
    p = assemble(src) if isinstance(src, str) else src
    return rc.rc_prove(rc.rc_load_program(p.bytecode), n, sizes, **kw)


@pytest.mark.parametrize("name,src,n,sizes,verdict,reason", [
    ("stencil", K.STENCIL, 1000, [1002, 1002], "NO_CONFLICT", None),
    ("stencil_full", K.STENCIL, 1 << 20, [(1 << 20) + 2] * 2, "NO_CONFLICT", None),
    ("tree", K.TREE, 1024, [1024], "NO_CONFLICT", None),
    ("tree_off_by_one", K.TREE_OFF_BY_ONE, 1024, [1024], "UNKNOWN", "OOB"),
    ("fig1", K.FIG1, 8, [8, 8, 8], "UNKNOWN", "OOB"),
    ("fig1_guarded", K.FIG1_GUARDED, 8, [8, 8, 8], "UNKNOWN", "RW"),
    ("fig2", K.FIG2, 2, [3, 1], "UNKNOWN", "RW"),
    ("K_c", K.BENIGN["K_c"], 256, [1, 256], "NORACE", None),
    ("K_tid", K.BENIGN["K_tid"], 256, [1, 256], "UNKNOWN", "WW"),
    ("K_B0", K.BENIGN["K_B0"], 256, [1, 256], "NORACE", None),
    ("K_Btid", K.BENIGN["K_Btid"], 256, [1, 256], "UNKNOWN", "WW"),
    ("K_last", K.BENIGN["K_last"], 256, [1, 256], "NORACE", None),
    ("K_inc", K.BENIGN["K_inc"], 256, [1, 256], "UNKNOWN", "RW"),
    ("private_only", K.PRIVATE_ONLY, 64, [4], "NO_CONFLICT", None),
])
def test_pins(rc, name, src, n, sizes, verdict, reason):
    r = prove(rc, src, n, sizes)
    assert (r.verdict, r.reason) == (verdict, reason), r


def test_fig1_interval_and_stencil_intervals(rc):
    """The RW race of Fig. 1 is in its second interval (after the barrier):
    the first interval is checked, the second stops the proof; the stencil
    checks all 9 intervals (8 barriers + the final one, App. A.5)."""
    r = prove(rc, K.FIG1_GUARDED, 8, [8, 8, 8])
    assert r.intervals == 1
    r = prove(rc, K.STENCIL, 64, [66, 66])
    assert r.intervals == 9


def test_small_shapes_decide_collisions(rc):
    """The prover decides over the concrete range: A[tid] := 0; A[tid+1]...
    written at distinct tids of one interval collide (tid i writes A[i+1],
    tid i+1 writes A[i+1]) unless n == 1."""
    src = """
.arrays A
    tid   r0
    const r1, 5
    st    A, r0, r1
    addi  r2, r0, 1
    st    A, r2, r0
    exit
"""
    assert prove(rc, src, 1, [2]).verdict == "NO_CONFLICT"
    r = prove(rc, src, 2, [3])
    assert (r.verdict, r.reason) == ("UNKNOWN", "WW")  # tid 0 writes A[1] := 0, tid 1 writes A[1] := 5
    # an index that runs off the array for the largest tid only
    assert prove(rc, src, 3, [3]).reason == "OOB"


def test_data_dependent_index_is_unknown(rc):
    src = """
.arrays A B
    tid   r0
    ld    r1, B, r0
    const r2, 1
    st    A, r1, r2
    exit
"""
    r = prove(rc, src, 4, [4, 4])
    assert (r.verdict, r.reason) == ("UNKNOWN", "DATA_INDEX")


def test_budget_is_unknown(rc):
    r = prove(rc, K.STENCIL, 1 << 16, [(1 << 16) + 2] * 2, budget=1000)
    assert (r.verdict, r.reason) == ("UNKNOWN", "BUDGET")


def _reports(prog, n, ins, fuel=64):
    return oracle.run(prog.bytecode, n, ins, fuel=fuel).report_tuples()


def test_soundness_against_the_oracle(rc):
    """Random kernels (the brute-force generator): NO_CONFLICT => the concrete
    checker reports nothing; NORACE => only WW_BENIGN, on random inputs with
    small value ranges (equal values by chance are frequent)."""
    rng = np.random.default_rng(2024)
    proved = {"NO_CONFLICT": 0, "NORACE": 0, "UNKNOWN": 0}
    for it in range(1500):
        n = int(rng.integers(1, 7))
        size = int(rng.integers(2, 7))
        p = K.random_tiny_kernel(rng, n_arrays=2, n_regs=4, n_commands=int(rng.integers(2, 8)), size=size)
        r = rc.rc_prove(rc.rc_load_program(p.bytecode), n, [size, size], fuel_per_interval=64)
        proved[r.verdict] += 1
        if r.verdict == "UNKNOWN":
            continue
        for trial in range(3):
            ins = [rng.integers(-2, 3, size=(2, size)).astype(np.int32) for _ in range(2)]
            kinds = {t[4] for t in _reports(p, n, ins)}
            if r.verdict == "NO_CONFLICT":
                assert not kinds, (it, r, kinds)
            else:
                assert kinds <= {2}, (it, r, kinds)
    # the prover is not vacuous on this generator
    assert proved["NO_CONFLICT"] > 100 and proved["NORACE"] > 10, proved


def test_norace_means_deterministic_shared_state(rc):
    """The paper's NoRace says the shared state at every barrier
    is deterministic: for proved kernels at n <= 3 every interval has exactly
    one reachable end heap over all interleavings."""
    from oracle import oracle as orc
    rng = np.random.default_rng(77)
    checked = 0
    for it in range(400):
        n = int(rng.integers(2, 4))
        size = int(rng.integers(2, 5))
        p = K.random_tiny_kernel(rng, n_arrays=2, n_regs=4, n_commands=int(rng.integers(2, 6)), size=size)
        r = rc.rc_prove(rc.rc_load_program(p.bytecode), n, [size, size], fuel_per_interval=64)
        if r.verdict == "UNKNOWN":
            continue
        ins = [rng.integers(-2, 3, size=size).astype(np.int32) for _ in range(2)]
        res = orc.run(p.bytecode, n, [x.reshape(1, -1) for x in ins], fuel=64, threads=1)
        for k in range(res.stats["intervals_max"]):
            reached, heap, regs, pc, st = orc.state_at(p.bytecode, n, ins, k, fuel=64)
            assert reached
            e = orc.enumerate_interval(p.bytecode, n, [size, size], heap, regs, pc, st, fuel=64,
                                       budget=2_000_000, reduced=True)
            assert e.complete
            assert len(set(e.heaps)) == 1, (it, r, k)
        checked += 1
    assert checked > 50


def test_invalid_arguments(rc):
    p = assemble(K.STENCIL)
    prog = rc.rc_load_program(p.bytecode)
    with pytest.raises(rc.RCError):
        rc.rc_prove(prog, 8, [10])  # n_arrays mismatch
    with pytest.raises(rc.RCError):
        rc.rc_prove(prog, 0, [10, 10])
