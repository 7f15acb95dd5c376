"""GPU interleaving explorer (rc_explore) against the
oracle's brute-force enumerator (oracle.c part 2).

Parity items, per explored interval:
  * the set of distinct end states (heap + every lane's pc, status and
    registers) equals the enumerator's, in both modes (all steps / shared
    accesses only);
  * with every instruction a step, the number of schedules equals the
    enumerator's count (and C(a+b, a) in the closed-form case);
  * n_differ > 0 iff the enumerator finds more than one end heap (the paper's
    race definition), and the witness schedule's end heap is a
    reachable one that differs from schedule 0's.
"""
import math

import numpy as np
import pytest

from workloads import inputs as I
from workloads import kernels as K
from workloads.asm import assemble

pytestmark = pytest.mark.gpu


def _explore(prog, n, sizes, heap, regs, pc, st, *, reduced, fuel=64, cap=0, max_len=256):
    import torch

    from paper_1308_3203_b200 import rc_explore
    end = 1 << 12
    while True:
        r = rc_explore(prog, n, torch.from_numpy(np.ascontiguousarray(heap, np.int32)).cuda(),
                       regs=torch.from_numpy(np.ascontiguousarray(regs, np.int32)).cuda(),
                       pc=torch.from_numpy(pc.astype(np.int32)).cuda(),
                       status=torch.from_numpy(st.astype(np.uint8)).cuda(), sizes=sizes, fuel=fuel,
                       index_end=end, reduced=reduced, cap=cap, max_len=max_len)
        if r.complete:
            return r
        assert end < (1 << 34), "schedule space too large for a test"
        end = max(2 * end, r.max_product)


def _rows(t):
    return {tuple(int(v) for v in row) for row in np.unique(t.cpu().numpy(), axis=0)} if t is not None else set()


def check_interval(orc, p, n, sizes, heap, regs, pc, st, *, full, fuel=64):
    """Compare the GPU explorer with the enumerator on one interval start state."""
    from paper_1308_3203_b200 import rc_load_program
    prog = rc_load_program(p.bytecode)
    e = orc.enumerate_interval(p.bytecode, n, sizes, heap, regs, pc, st, fuel=fuel)
    assert e.complete
    cells = int(sum(sizes))
    cap = 1 << 21
    modes = [True, False] if (full and e.n_schedules <= 1_000_000) else [True]
    for reduced in modes:
        r = _explore(prog, n, sizes, heap, regs, pc, st, reduced=reduced, fuel=fuel, cap=cap)
        rows = _rows(r.terminals)
        if r.n_schedules <= cap:
            assert rows == set(e.lanes), f"end states differ (reduced={reduced})"
        else:
            assert rows <= set(e.lanes)
        if not reduced:
            assert r.n_schedules == e.n_schedules
        assert (r.n_differ > 0) == (len(e.heaps) > 1)
        if r.witness is not None:
            # replay the witness and schedule 0 alone: their end heaps differ, both reachable
            w = _one(prog, n, sizes, heap, regs, pc, st, r.witness, reduced, fuel)
            z = _one(prog, n, sizes, heap, regs, pc, st, 0, reduced, fuel)
            assert w[:cells] != z[:cells] and w[:cells] in e.heaps and z[:cells] in e.heaps
            assert 0 < len(r.witness_sched) and all(0 <= t < n for t in r.witness_sched)
    return e


def _one(prog, n, sizes, heap, regs, pc, st, index, reduced, fuel):
    import torch

    from paper_1308_3203_b200 import rc_explore
    r = rc_explore(prog, n, torch.from_numpy(np.ascontiguousarray(heap, np.int32)).cuda(),
                   regs=torch.from_numpy(np.ascontiguousarray(regs, np.int32)).cuda(),
                   pc=torch.from_numpy(pc.astype(np.int32)).cuda(), status=torch.from_numpy(st.astype(np.uint8)).cuda(),
                   sizes=sizes, fuel=fuel, index_begin=index, index_end=index + 1, reduced=reduced, cap=1)
    assert r.n_schedules == 1
    return tuple(int(v) for v in r.terminals[0].cpu().numpy())


def test_explore_schedule_count_closed_form(oracle_lib):
    """Two work-items with a and b private steps: C(a+b, a) schedules, one end
    state; shared-access-only scheduling: exactly 1."""
    from paper_1308_3203_b200 import rc_load_program
    for a in range(1, 6):
        for b in range(1, 6):
            lines = [".arrays A", " tid r0", " br r0, t1, t0"]
            lines += ["t0:"] + [f" addi r1, r1, {i + 1}" for i in range(a - 1)] + [" exit"]
            lines += ["t1:"] + [f" addi r2, r2, {i + 1}" for i in range(b - 1)] + [" exit"]
            p = assemble("\n".join(lines))
            pc = np.array([p.labels["t0"], p.labels["t1"]], np.uint32)
            regs = np.zeros((2, p.n_regs), np.int32)
            regs[1, 0] = 1
            st = np.zeros(2, np.uint8)
            prog = rc_load_program(p.bytecode)
            r = _explore(prog, 2, [1], np.zeros(1, np.int32), regs, pc, st, reduced=False, cap=64)
            assert r.n_schedules == math.comb(a + b, a) and r.n_differ == 0 and r.witness is None
            assert len(_rows(r.terminals)) == 1
            r = _explore(prog, 2, [1], np.zeros(1, np.int32), regs, pc, st, reduced=True)
            assert r.n_schedules == 1


def test_explore_fig1(oracle_lib):
    """App. A.1, n = 4: interval 1 reaches R = [100,84,206,103] and
    [100,412,206,103]; the explorer finds both and a witness."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fig1.json")))["bruteforce_n4"]
    p = K.program(K.FIG1_GUARDED)
    ins = [np.array(g["inputs"][a], np.int32) for a in ("A", "B", "R")]
    for k in (0, 1):
        reached, heap, regs, pc, st = oracle_lib.state_at(p.bytecode, 4, ins, k)
        e = check_interval(oracle_lib, p, 4, [4, 4, 4], heap, regs, pc, st, full=False)
    assert sorted({h[8:12] for h in e.heaps}) == sorted(tuple(x) for x in g["interval1_F_R"])


@pytest.mark.parametrize("A2", [5, 0])
def test_explore_fig2(oracle_lib, A2):
    """g in {0, 1} for A[2] != 0, only 1 for A[2] = 0."""
    p = K.program(K.FIG2)
    ins = [np.array([7, 9, A2], np.int32), np.array([42], np.int32)]
    for k in (0, 1):
        reached, heap, regs, pc, st = oracle_lib.state_at(p.bytecode, 2, ins, k)
        if not reached:
            continue
        check_interval(oracle_lib, p, 2, [3, 1], heap, regs, pc, st, full=True)


@pytest.mark.parametrize("name", list(K.BENIGN))
def test_explore_benign_suite(oracle_lib, name):
    """App. A.3 at n = 2..4 (all steps at n = 2)."""
    p = K.program(K.BENIGN[name])
    for n in (2, 3, 4):
        for B in (np.full(n, 3, np.int32), np.arange(n, dtype=np.int32) % 2):
            ins = [np.array([40], np.int32), B]
            reached, heap, regs, pc, st = oracle_lib.state_at(p.bytecode, n, ins, 0)
            check_interval(oracle_lib, p, n, [1, n], heap, regs, pc, st, full=(n == 2))


def test_explore_tree_and_stencil(oracle_lib):
    """Config 3 / config 5 shapes at n = 4 / 3, every interval."""
    cases = []
    for src in (K.TREE, K.TREE_OFF_BY_ONE):
        A = np.random.default_rng(3).integers(-5, 5, 4).astype(np.int32)
        cases.append((K.program(src), 4, [A]))
    A, B = I.cfg5_inputs(0, 1, 3)
    cases.append((K.program(K.STENCIL), 3, [A[0], B[0]]))
    for p, n, ins in cases:
        sizes = [int(x.shape[-1]) for x in ins]
        res = oracle_lib.run(p.bytecode, n, [x.reshape(1, -1) for x in ins], fuel=64, threads=1)
        for k in range(res.stats["intervals_max"]):
            reached, heap, regs, pc, st = oracle_lib.state_at(p.bytecode, n, ins, k, fuel=64)
            check_interval(oracle_lib, p, n, sizes, heap, regs, pc, st, full=False)


def test_explore_random_tiny_kernels(oracle_lib):
    """Random tiny kernels (n <= 3, arrays of 3): both modes against the enumerator."""
    rng = np.random.default_rng(8_3203)
    racy = 0
    for it in range(150):
        n = int(rng.integers(2, 4))
        p = K.random_tiny_kernel(rng, n_arrays=2, n_regs=4, n_commands=int(rng.integers(3, 7)), size=3)
        ins = I.tiny_inputs(rng, 2, 3)
        reached, heap, regs, pc, st = oracle_lib.state_at(p.bytecode, n, ins, 0, fuel=64)
        e = check_interval(oracle_lib, p, n, [3, 3], heap, regs, pc, st, full=(n == 2), fuel=64)
        racy += len(e.heaps) > 1
    assert racy > 10  # the family does produce non-deterministic intervals


def test_explore_global_scratch_path(oracle_lib, monkeypatch):
    """State rows in the global scratch instead of shared memory (the path of
    large rows; forced by a test hook): the same end states and counts."""
    monkeypatch.setenv("RC_DEBUG_EXPLORE_GLOBAL", "1")
    p = K.program(K.FIG2)
    ins = [np.array([7, 9, 5], np.int32), np.array([42], np.int32)]
    reached, heap, regs, pc, st = oracle_lib.state_at(p.bytecode, 2, ins, 1)
    check_interval(oracle_lib, p, 2, [3, 1], heap, regs, pc, st, full=True)
    p = K.program(K.BENIGN["K_inc"])
    reached, heap, regs, pc, st = oracle_lib.state_at(p.bytecode, 4, [np.array([40], np.int32), np.zeros(4, np.int32)], 0)
    check_interval(oracle_lib, p, 4, [1, 4], heap, regs, pc, st, full=False)


def test_explore_edge_cases(oracle_lib):
    """n = 1 (one schedule), no runnable work-item (the empty schedule), and
    index sub-ranges: disjoint ranges add up to the whole exploration."""
    import torch

    from paper_1308_3203_b200 import rc_explore, rc_load_program
    p = K.program(K.BENIGN["K_inc"])
    prog = rc_load_program(p.bytecode)

    def state(n):
        _, heap, regs, pc, st = oracle_lib.state_at(p.bytecode, n, [np.array([40], np.int32), np.zeros(n, np.int32)], 0)
        return (torch.from_numpy(heap.astype(np.int32)).cuda(), torch.from_numpy(regs).cuda(),
                torch.from_numpy(pc.astype(np.int32)).cuda(), torch.from_numpy(st).cuda())

    heap, regs, pc, st = state(1)
    for red in (True, False):
        r = rc_explore(prog, 1, heap, regs=regs, pc=pc, status=st, sizes=[1, 1], index_end=8, reduced=red, cap=8)
        assert r.complete and r.n_schedules == 1 and r.n_differ == 0 and r.witness is None
        assert int(r.terminals[0, 0]) == 41  # A[0] + 1
    heap, regs, pc, st = state(3)
    waiting = torch.ones_like(st)  # every work-item suspended at a barrier: nothing steps
    r = rc_explore(prog, 3, heap, regs=regs, pc=pc, status=waiting, sizes=[1, 3], index_end=4, cap=4)
    assert r.complete and r.n_schedules == 1 and r.max_product == 1
    assert r.terminals[0].cpu().tolist()[:4] == heap.cpu().tolist()  # the heap is untouched
    whole = rc_explore(prog, 3, heap, regs=regs, pc=pc, status=st, sizes=[1, 3], index_end=1 << 12)
    assert whole.complete and whole.n_schedules == 90  # 6! / 2^3 interleavings of 3 x (LD, ST)
    parts = [rc_explore(prog, 3, heap, regs=regs, pc=pc, status=st, sizes=[1, 3], index_begin=a, index_end=b)
             for a, b in ((0, 100), (100, 1000), (1000, 1 << 12))]
    assert sum(x.n_schedules for x in parts) == 90 and sum(x.n_differ for x in parts) == whole.n_differ
    assert min(x.witness for x in parts if x.witness is not None) == whole.witness
    assert not parts[1].complete  # only a range that starts at 0 can be complete
    empty = rc_explore(prog, 3, heap, regs=regs, pc=pc, status=st, sizes=[1, 3], index_begin=0, index_end=0)
    assert not empty.complete and empty.n_schedules == 0  # nothing examined: schedule 0 exists but was not seen
