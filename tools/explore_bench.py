"""Throughput of the GPU interleaving explorer (rc_explore, SURVEY.md §8(f)
row 2) beside the oracle's enumerator (dev tool; prints one JSON line per
workload).

Workloads (seeded): K_inc (App. A.3 lost update, 2 accesses per work-item)
at n = 5 / 6 and guarded Fig. 1 interval 1 at n = 4, shared-access
scheduling (RC_EXPLORE_REDUCED).  GPU time = CUDA events around one complete
rc_explore call, best of 5 (after one warm-up call; the call includes its
device allocations and the start-state upload); the first case schedules every
instruction, as the un-memoised oracle walk does, the others only the
shared accesses.  The oracle legs: the memoised
enumerator over the whole interval, and the un-memoised walk (every schedule
visited, like the GPU) on a bounded budget.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as orc  # noqa: E402
from paper_1308_3203_b200 import rc_explore, rc_load_program  # noqa: E402
from workloads import kernels as K  # noqa: E402


def explore_all(prog, n, sizes, heap, regs, pc, st, reduced=True):
    end = 1 << 16
    while True:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        r = rc_explore(prog, n, heap, regs=regs, pc=pc, status=st, sizes=sizes, index_end=end, reduced=reduced)
        ev1.record()
        torch.cuda.synchronize()
        if r.complete:
            return r, end, ev0.elapsed_time(ev1)
        end = max(2 * end, r.max_product)


def case(name, p, n, ins, k, reduced=True):
    sizes = [int(x.shape[-1]) for x in ins]
    reached, heap, regs, pc, st = orc.state_at(p.bytecode, n, ins, k)
    prog = rc_load_program(p.bytecode)
    d = dict(heap=torch.from_numpy(heap.astype(np.int32)).cuda(), regs=torch.from_numpy(regs).cuda(),
             pc=torch.from_numpy(pc.astype(np.int32)).cuda(), st=torch.from_numpy(st).cuda())
    explore_all(prog, n, sizes, d["heap"], d["regs"], d["pc"], d["st"], reduced)  # warm-up
    runs = [explore_all(prog, n, sizes, d["heap"], d["regs"], d["pc"], d["st"], reduced) for _ in range(5)]
    r, end, ms = min(runs, key=lambda x: x[2])  # best of 5 complete calls
    t0 = time.perf_counter()
    e = orc.enumerate_interval(p.bytecode, n, sizes, heap, regs, pc, st)
    t_memo = time.perf_counter() - t0
    budget = 2_000_000
    t0 = time.perf_counter()
    e2 = orc.enumerate_interval(p.bytecode, n, sizes, heap, regs, pc, st, memo=False, budget=budget)
    t_walk = time.perf_counter() - t0
    print(json.dumps({
        "workload": name, "n": n, "mode": "shared accesses" if reduced else "every instruction", "interval": k, "schedules": r.n_schedules, "end_heaps_differ": r.n_differ,
        "indices": end, "valid_fraction": r.n_schedules / end, "gpu_ms": round(ms, 3),
        "gpu_schedules_per_s": r.n_schedules / (ms / 1e3), "gpu_indices_per_s": end / (ms / 1e3),
        "oracle_memo_s": round(t_memo, 3), "oracle_memo_states_distinct_heaps": len(e.heaps),
        "oracle_walk_schedules_per_s": (e2.n_schedules if e2.complete else budget) / t_walk,
        "oracle_walk_note": "full-step schedules (every instruction a step), 1 thread",
    }))


def main():
    assert torch.cuda.is_available()
    # every instruction a step: the same schedules the un-memoised oracle walk visits
    case("K_inc n=3", K.program(K.BENIGN["K_inc"]), 3, [np.array([40], np.int32), np.zeros(3, np.int32)], 0, False)
    for n in (5, 6):
        case(f"K_inc n={n}", K.program(K.BENIGN["K_inc"]), n, [np.array([40], np.int32), np.zeros(n, np.int32)], 0)
    g = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "fig1.json")))["bruteforce_n4"]
    ins = [np.array(g["inputs"][a], np.int32) for a in ("A", "B", "R")]
    case("fig1 guarded n=4", K.program(K.FIG1_GUARDED), 4, ins, 1)


if __name__ == "__main__":
    main()
