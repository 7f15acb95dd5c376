"""Pins of the oracle's RW value classification (SURVEY.md §8(f) row 1,
DESIGN.md §3 reading L19).

The classification re-runs an interval with an RW report under a second
visibility — reads of the RW-flagged cells see the value the canonical run
committed (writers first) — commits that run's writes onto the
interval-start heap and compares the two committed heaps.  RW reports get
flag bit 4 (0x10, equal heaps: the race does not change the state for this
input) or bit 5 (0x20, the committed state depends on the read values).

Expected values are hand-derived closed forms (lost update, unused reads,
Fig. 1's doubling chain), never the oracle's own output.
"""
import json
import os

import numpy as np

from workloads import inputs as I
from workloads import kernels as K
from workloads.asm import assemble

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RW, WWB = 1, 2
NOTID = 0xFFFFFFFF


def rw_flags(res):
    return [t[7] for t in res.report_tuples() if t[4] == RW]


def test_lost_update_is_value_dependent(oracle_lib):
    """K_inc (A[0] := A[0] + 1 by every work-item), n = 4, A[0] = 10: the
    canonical run commits 11; with writers first every read sees 11 and the
    commit is 12 -> bit 5.  The WW report (all wrote 11: benign) is untouched."""
    p = K.program(K.BENIGN["K_inc"])
    ins = [np.array([[10]], np.int32), np.zeros((1, 4), np.int32)]
    r = oracle_lib.run(p.bytecode, 4, ins, classify_rw=True)
    assert r.report_tuples() == [(0, 0, 0, 0, RW, 0, 1, 15 | 0x20), (0, 0, 0, 0, WWB, 0, 1, 15)]
    assert r.final[0][0, 0] == 11  # the canonical commit stands
    r0 = oracle_lib.run(p.bytecode, 4, ins)
    assert r0.report_tuples() == [(0, 0, 0, 0, RW, 0, 1, 15), (0, 0, 0, 0, WWB, 0, 1, 15)]


def test_unused_read_is_benign(oracle_lib):
    """Every work-item reads A[0] and writes the constant 5 to it: the read
    value feeds nothing, so both runs commit 5 -> bit 4."""
    src = ".arrays A\n const r0, 0\n ld r1, A, r0\n const r2, 5\n st A, r0, r2\n exit\n"
    p = assemble(src)
    for a0 in (9, 5):
        r = oracle_lib.run(p.bytecode, 3, [np.array([[a0]], np.int32)], classify_rw=True)
        assert rw_flags(r) == [15 | 0x10]
        assert r.final[0][0, 0] == 5


def test_neighbour_reads(oracle_lib):
    """Work-item t reads A[t+1] and writes A[t] := t (size n+1): RW on
    A[1..n-1].  Unused read -> bit 4 on all of them; feeding the read into
    B[t] := A[t+1] makes B depend on it (A[t+1] = c+t+1 before, t+1 after)
    -> bit 5."""
    n = 6
    base = ".arrays A B\n tid r0\n addi r1, r0, 1\n ld r2, A, r1\n st A, r0, r0\n"
    A = (100 + np.arange(n + 1, dtype=np.int32))[None, :]
    B = np.zeros((1, n), np.int32)
    p = assemble(base + " exit\n")
    r = oracle_lib.run(p.bytecode, n, [A, B], classify_rw=True)
    assert len(rw_flags(r)) == n - 1 and all(f & 0x30 == 0x10 for f in rw_flags(r))
    p = assemble(base + " st B, r0, r2\n exit\n")
    r = oracle_lib.run(p.bytecode, n, [A, B], classify_rw=True)
    assert len(rw_flags(r)) == n - 1 and all(f & 0x30 == 0x20 for f in rw_flags(r))
    assert r.final[1][0].tolist() == [101, 102, 103, 104, 105, 106]  # canonical: interval-start values


def test_fig1_doubling_chain(oracle_lib):
    """PAPER.md:62-74 (App. A.1): interval 1 computes R[t] := 2 R[t+1] from
    R[t] = 11t + 20; with writers first R[t+1] is already doubled, so the
    committed R changes -> bit 5 on every RW report of interval 1."""
    with open(os.path.join(GOLD, "fig1.json")) as f:
        g = json.load(f)
    p = K.program(K.FIG1)
    r = oracle_lib.run(p.bytecode, 8, I.cfg1_inputs(), classify_rw=True)
    exp = []
    for x in g["reports_verbatim"]:
        arr = p.arrays.index(x["array"])
        fl = x.get("flags", 0) | (0x20 if x["kind"] == "RW" else 0)
        exp.append((0, x["interval"], arr, x["index"], {"RW": 1, "OOB": 4}[x["kind"]], x["tid1"],
                    x.get("tid2", NOTID), fl))
    assert r.report_tuples() == exp
    assert r.final[2][0].tolist() == g["final_R"]


def test_classification_changes_nothing_else(oracle_lib):
    """With classification on, reports differ only in bits 4/5 of RW reports
    (exactly one of them set on each), and final heaps and statistics are
    unchanged, over random small kernels and the configuration kernels."""
    rng = np.random.default_rng(5)
    cases = [(K.TREE_OFF_BY_ONE, 64, I.cfg3_inputs(0, 3, 64)), (K.STENCIL, 50, I.cfg5_inputs(0, 2, 50))]
    for name in K.BENIGN:
        cases.append((K.BENIGN[name], 16, I.cfg2_inputs(0, 4, 16)))
    for _ in range(200):
        n = int(rng.integers(1, 9))
        pr = K.random_tiny_kernel(rng, n_arrays=2, n_regs=5, n_commands=int(rng.integers(3, 12)), size=5)
        ins = [rng.integers(-3, 4, size=(2, 5)).astype(np.int32) for _ in range(2)]
        cases.append((pr, n, ins))
    for src, n, ins in cases:
        p = K.program(src) if isinstance(src, str) else src
        a = oracle_lib.run(p.bytecode, n, ins, fuel=500)
        b = oracle_lib.run(p.bytecode, n, ins, fuel=500, classify_rw=True)
        ta, tb = a.report_tuples(), b.report_tuples()
        assert len(ta) == len(tb)
        for x, y in zip(ta, tb):
            assert x[:7] == y[:7] and x[7] == (y[7] & ~0x30)
            assert (y[7] & 0x30) in ((0x10, 0x20) if y[4] == RW else (0,))
        for fa, fb in zip(a.final, b.final):
            assert np.array_equal(fa, fb)
        assert a.stats == b.stats
