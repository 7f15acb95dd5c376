"""Brute-force interleaving checks tying the canonical oracle to the paper.

The enumerator (oracle.c part 2) implements the paper's global semantics
(PAPER.md:204-227): one thread steps at a time on a shared heap with
immediate visibility.  For each barrier interval k of a small run it explores
every interleaving from the canonical interval-start state and collects F_k,
the set of reachable end-of-interval states.  Invariants:

  I1  no RW report in k  =>  (|F_k| > 1  <=>  some WW_NONBENIGN report in k)
  I2  |F_k| > 1          =>  some RW or WW_NONBENIGN report in k
  I3  no report of kind 1-3 in k  =>  F_k = {canonical end state} (heap and lanes)
  I4  no RW report in k  =>  canonical committed heap is in F_k

I1 is north_star's "a non-benign race exists iff some interleaving yields a
different final heap", which holds exactly for RW-free intervals; App. A.2
and A.3 (K_inc) show that under RW only I2 holds.
"""
import json
import math
import os

import numpy as np
import pytest

from workloads import inputs as I
from workloads import kernels as K
from workloads.asm import assemble

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def check_intervals(orc, prog, n, inputs, fuel=64, budget=3_000_000, reduced=False):
    """Run the canonical oracle on one instance and check I1-I4 for every
    interval against exhaustive enumeration.  Returns per-interval |F|.
    reduced: enumerate with only LD / ST as scheduling points (the same
    terminal set, checked against the full enumeration below)."""
    sizes = [int(x.shape[-1]) for x in inputs]
    ins2 = [x.reshape(1, -1) for x in inputs]
    res = orc.run(prog.bytecode, n, ins2, fuel=fuel, threads=1)
    reps = res.report_tuples()
    n_int = res.stats["intervals_max"]
    out = []
    for k in range(n_int):
        reached, heap, regs, pc, st = orc.state_at(prog.bytecode, n, [x.reshape(-1) for x in inputs], k, fuel=fuel)
        assert reached
        e = orc.enumerate_interval(prog.bytecode, n, sizes, heap, regs, pc, st, fuel=fuel, budget=budget,
                                   reduced=reduced)
        assert e.complete, "enumeration budget exceeded"
        kinds = {t[4] for t in reps if t[1] == k}
        F = set(e.heaps)
        has_rw, has_wwn = 1 in kinds, 3 in kinds
        # canonical end of interval k = start of k+1 (or the final state)
        _, heap1, regs1, pc1, st1 = orc.state_at(prog.bytecode, n, [x.reshape(-1) for x in inputs], k + 1, fuel=fuel)
        canon_heap = tuple(int(x) for x in heap1)
        if len(F) > 1:
            assert has_rw or has_wwn, f"I2 violated at interval {k}"
        if not has_rw:
            assert (len(F) > 1) == has_wwn, f"I1 violated at interval {k}"
            assert canon_heap in F, f"I4 violated at interval {k}"
        if not (kinds & {1, 2, 3}):
            assert F == {canon_heap}, f"I3 (heap) violated at interval {k}"
            # lanes: the enumerator leaves suspended lanes WAITING; the canonical
            # state at k+1 has released them (WAITING -> RUNNING)
            cells = len(canon_heap)
            lw = 4 + regs.shape[1]
            lane_sets = set()
            for row in e.lanes:
                lanes = []
                for t in range(n):
                    L = row[cells + t * lw: cells + (t + 1) * lw]
                    stt = 0 if L[1] == 1 else L[1]
                    lanes.append((L[0], stt) + tuple(L[4:]))
                lane_sets.add(tuple(lanes))
            canon_lanes = tuple((int(pc1[t]), int(st1[t])) + tuple(int(x) for x in regs1[t]) for t in range(n))
            assert lane_sets == {canon_lanes}, f"I3 (lanes) violated at interval {k}"
        out.append(len(F))
    return out


def test_fig1_bruteforce(oracle_lib):
    """App. A.1 brute force: n=4, arrays of 4, guarded Fig. 1; interval 1 has
    F = {[100,84,206,103], [100,412,206,103]} and the canonical heap in F."""
    g = json.load(open(os.path.join(GOLD, "fig1.json")))["bruteforce_n4"]
    p = K.program(K.FIG1_GUARDED)
    ins = [np.array(g["inputs"][a], np.int32) for a in ("A", "B", "R")]
    sizes = [4, 4, 4]
    reached, heap, regs, pc, st = oracle_lib.state_at(p.bytecode, 4, ins, 1)
    e = oracle_lib.enumerate_interval(p.bytecode, 4, sizes, heap, regs, pc, st)
    Rs = sorted({h[8:12] for h in e.heaps})
    assert Rs == sorted(tuple(x) for x in g["interval1_F_R"])
    r = oracle_lib.run(p.bytecode, 4, [x.reshape(1, -1) for x in ins])
    assert r.final[2][0].tolist() == g["canonical_R"]
    assert check_intervals(oracle_lib, p, 4, ins) == [1, 2, 1][:r.stats["intervals_max"]]


@pytest.mark.parametrize("A2,expect_G", [(5, [0, 1]), (0, [1])])
def test_fig2_bruteforce(oracle_lib, A2, expect_G):
    """PAPER.md:468 'g can in practice have the value 0 or the value 1' —
    true for A[2]=5; for A[2]=0 only g=1 is reachable although RW is reported."""
    p = K.program(K.FIG2)
    ins = [np.array([7, 9, A2], np.int32), np.array([42], np.int32)]
    reached, heap, regs, pc, st = oracle_lib.state_at(p.bytecode, 2, ins, 1)
    e = oracle_lib.enumerate_interval(p.bytecode, 2, [3, 1], heap, regs, pc, st)
    assert sorted({h[3] for h in e.heaps}) == expect_G
    check_intervals(oracle_lib, p, 2, ins)


@pytest.mark.parametrize("name", list(K.BENIGN))
@pytest.mark.parametrize("n", [2, 3, 4])
def test_benign_bruteforce(oracle_lib, name, n):
    """App. A.3 at n <= 4: K_c, K_B0, K_last give |F| = 1; K_tid gives |F| = n;
    K_Btid gives |F| = number of distinct B values; K_inc (lost updates) gives
    F = {A0+1, ..., A0+n}."""
    p = K.program(K.BENIGN[name])
    for B in (np.full(n, 3, np.int32), np.arange(n, dtype=np.int32) % 2):
        ins = [np.array([40], np.int32), B]
        F = check_intervals(oracle_lib, p, n, ins)
        if name in ("K_c", "K_B0", "K_last"):
            assert F == [1]
        elif name == "K_tid":
            assert F == [n]
        elif name == "K_Btid":
            assert F == [len(set(B.tolist()))]
        elif name == "K_inc":
            # every schedule increments at least once and at most n times
            reached, heap, regs, pc, st = oracle_lib.state_at(p.bytecode, n, ins, 0)
            e = oracle_lib.enumerate_interval(p.bytecode, n, [1, n], heap, regs, pc, st)
            assert sorted(h[0] for h in e.heaps) == list(range(41, 41 + n))


def test_tree_reduction_bruteforce(oracle_lib):
    """Config 3 shape at n=4: race-free reduction has |F_k| = 1 every interval;
    the off-by-one variant is RW-racy but I1-I4 still hold."""
    for src in (K.TREE, K.TREE_OFF_BY_ONE):
        p = K.program(src)
        for seed in range(3):
            A = np.random.default_rng(seed).integers(-5, 5, 4).astype(np.int32)
            F = check_intervals(oracle_lib, p, 4, [A])
            if src is K.TREE:
                assert all(f == 1 for f in F)


def test_stencil_bruteforce(oracle_lib):
    p = K.program(K.STENCIL)
    A, B = I.cfg5_inputs(0, 1, 3)
    F = check_intervals(oracle_lib, p, 3, [A[0], B[0]], budget=10_000_000)
    assert all(f == 1 for f in F)


@pytest.mark.parametrize("a,b", [(a, b) for a in range(1, 5) for b in range(1, 5)])
def test_schedule_count(oracle_lib, a, b):
    """two threads with a and b steps (private commands, no
    pruning) have exactly C(a+b, a) maximal interleavings, counted without
    memoisation; memoised counting gives the same number."""
    # thread 0 runs a instructions (incl. EXIT), thread 1 runs b
    lines = [".arrays A", " tid r0", " br r0, t1, t0"]
    lines += ["t0:"] + [f" addi r1, r1, {i + 1}" for i in range(a - 1)] + [" exit"]
    lines += ["t1:"] + [f" addi r2, r2, {i + 1}" for i in range(b - 1)] + [" exit"]
    p = assemble("\n".join(lines))
    # start both threads after the branch: pc of t0 / t1
    pc = np.array([p.labels["t0"], p.labels["t1"]], np.uint32)
    regs = np.zeros((2, p.n_regs), np.int32)
    regs[1, 0] = 1
    st = np.zeros(2, np.uint8)
    e0 = oracle_lib.enumerate_interval(p.bytecode, 2, [1], np.zeros(1, np.int32), regs, pc, st, memo=False)
    e1 = oracle_lib.enumerate_interval(p.bytecode, 2, [1], np.zeros(1, np.int32), regs, pc, st, memo=True)
    assert e0.n_schedules == math.comb(a + b, a) == e1.n_schedules
    assert len(e0.lanes) == 1  # private-only: one end state


def _tiny_case(i):
    """Random tiny kernel #i and its inputs: n in {2, 3, 4} work-items, two
    arrays of 3, 3-6 commands (full ALU, barriers, forward branches)."""
    rng = np.random.default_rng(np.random.SeedSequence([1308_3203, i]))
    n = int(rng.integers(2, 5))
    p = K.random_tiny_kernel(rng, n_arrays=2, n_regs=4, n_commands=int(rng.integers(3, 7)), size=3)
    ins = I.tiny_inputs(rng, 2, 3)
    return n, p, [x[0] for x in ins]


def _tiny_chunk(lo, hi):
    import oracle
    intervals = racy = 0
    by_n = [0, 0, 0, 0, 0]
    for i in range(lo, hi):
        n, p, ins = _tiny_case(i)
        try:
            F = check_intervals(oracle, p, n, ins, reduced=True)
        except AssertionError as ex:
            raise AssertionError(f"kernel #{i} (n={n}): {ex}\n{p.source}") from None
        intervals += len(F)
        racy += sum(f > 1 for f in F)
        by_n[n] += 1
    return intervals, racy, by_n


N_RANDOM_KERNELS = 12_000


def test_random_tiny_kernels(oracle_lib):
    """I1-I4 on 12 000 random tiny kernels at n <= 4 (>= 10^4),
    enumerated with only the shared accesses as scheduling points (pinned
    against the full enumeration by test_reduced_enumeration_same_terminals).
    Chunks run in forked worker processes (the oracle is a C library)."""
    import concurrent.futures as cf
    import multiprocessing as mp
    workers = max(1, min(len(os.sched_getaffinity(0)), 16))
    step = 250
    chunks = [(lo, min(lo + step, N_RANDOM_KERNELS)) for lo in range(0, N_RANDOM_KERNELS, step)]
    tot = racy = 0
    by_n = [0] * 5
    with cf.ProcessPoolExecutor(workers, mp_context=mp.get_context("fork")) as ex:
        for a, b, c in ex.map(_tiny_chunk, *zip(*chunks)):
            tot += a
            racy += b
            by_n = [x + y for x, y in zip(by_n, c)]
    assert sum(by_n) == N_RANDOM_KERNELS and min(by_n[2:]) > 3000  # every n in {2, 3, 4} well covered
    assert tot > N_RANDOM_KERNELS and racy > 500  # the generator does produce non-determinism


def test_reduced_enumeration_same_terminals(oracle_lib):
    """The reduced enumeration (only LD / ST interleave; every other step
    touches only its own thread's state, and commutes with
    the others) reaches exactly the terminal states (heap and every lane) of
    the full enumeration of PAPER.md:204-227, on the App. A kernels and 600
    random tiny kernels at n <= 3, every interval."""
    cases = [(K.program(K.FIG1_GUARDED), 4, [np.array([1, 2, 3, 4], np.int32), np.array([10, 20, 30, 40], np.int32),
                                               np.array([100, 101, 102, 103], np.int32)]),
             (K.program(K.FIG2), 2, [np.array([7, 9, 5], np.int32), np.array([42], np.int32)]),
             (K.program(K.BENIGN["K_inc"]), 3, [np.array([40], np.int32), np.zeros(3, np.int32)])]
    for i in range(600):
        rng = np.random.default_rng(np.random.SeedSequence([0xE4E4, i]))
        n = int(rng.integers(2, 4))
        p = K.random_tiny_kernel(rng, n_arrays=2, n_regs=4, n_commands=int(rng.integers(3, 7)), size=3)
        cases.append((p, n, [x[0] for x in I.tiny_inputs(rng, 2, 3)]))
    fewer = 0
    for p, n, ins in cases:
        sizes = [int(x.shape[-1]) for x in ins]
        k = 0
        while True:
            reached, heap, regs, pc, st = oracle_lib.state_at(p.bytecode, n, ins, k, fuel=64)
            if not reached:
                break
            full = oracle_lib.enumerate_interval(p.bytecode, n, sizes, heap, regs, pc, st, fuel=64)
            red = oracle_lib.enumerate_interval(p.bytecode, n, sizes, heap, regs, pc, st, fuel=64, reduced=True)
            assert full.complete and red.complete
            assert red.lanes == full.lanes, (k, p.source)
            assert red.n_schedules <= full.n_schedules
            fewer += red.n_schedules < full.n_schedules
            k += 1
    assert fewer > 100
