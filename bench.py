#!/usr/bin/env python
"""Benchmark of the race-checking hot path.

One step = one rc_run over the whole workload (all §8(a) rows: heap init,
every barrier interval's interpretation, write-set filter, grouping of the
log by cell (bucket scatter), per-bucket sort + detect + commit,
boundary bookkeeping, report finalize, report copy-out) plus, at N>1, the NCCL
report gather.  Default workload = BASELINE config 5 (3-point stencil,
2^20 work-items x 512 instances, 8 barrier intervals), STRONG scaling as
SURVEY.md §8(e) defines it: the 512 instances are split over the N ranks
(512/N each, contiguous shards).  Inputs (4.3 GB in all) are far larger than
the 126 MB L2, so no explicit flush is needed for the main line; the
secondary config-3 line flushes L2 before every timed step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0 (contract in the task statement / DESIGN.md §6).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from workloads import inputs as I  # noqa: E402
from workloads import kernels as K  # noqa: E402

# total = instances of the BASELINE configuration; strong scaling splits them
# over the ranks, weak scaling gives every rank `total` instances
WORKLOADS = {
    "cfg5": dict(name="config5: 3-point stencil, 2^20 work-items x 512 instances, 8 barriers",
                 n=1 << 20, total=512, src=lambda: K.program(K.STENCIL),
                 gen=lambda lo, hi, n: I.cfg5_inputs(lo, hi, n)),
    "cfg4": dict(name="config4: random straight-line stencil kernel (seed 0), 65536 work-items x 4096 instances",
                 n=65536, total=4096, src=lambda: K.random_stencil_kernel(0),
                 gen=lambda lo, hi, n: I.cfg4_inputs(lo, hi, n)),
    "cfg3": dict(name="config3: race-free tree reduction, 1024 work-items x 16384 instances, 11 intervals",
                 n=1024, total=16384, src=lambda: K.program(K.TREE),
                 gen=lambda lo, hi, n: I.cfg3_inputs(lo, hi, n)),
    "cfg3off": dict(name="config3: off-by-one tree reduction (1 OOB + 9 RW per instance), 1024 work-items x 16384 "
                         "instances", n=1024, total=16384, src=lambda: K.program(K.TREE_OFF_BY_ONE),
                    gen=lambda lo, hi, n: I.cfg3_inputs(lo, hi, n)),
}
METRIC = "checked memory accesses/s"
UNIT = "Gaccess/s"


def cub_baseline():
    """CUB's device radix sort on the same keys (7.3 M records, 24 cell bits,
    as in one config-5 interval), from the committed tools/cubbench.cu run."""
    path = os.path.join(ROOT, "profiles", "r01_sort_vs_cub.txt")
    if not os.path.exists(path):
        return None
    ours = cub = None
    for line in open(path):
        if "n=7340032" in line and "pattern=stencil" in line:
            gbs = float(line.split("->")[1].split("GB/s")[0])
            if line.startswith("CUB"):
                cub = gbs
            else:
                ours = gbs
    if cub is None:
        return None
    return {"kernel": "cub::DeviceRadixSort::SortKeys (CUB 2.8.2), same u64 records and 24 cell bits",
            "GBps": cub, "this_sort_GBps": ours, "records": 7340032, "source": "profiles/r01_sort_vs_cub.txt"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampling during the timed region (recipe's clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev = dev
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            time.sleep(0.25)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) != 6:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[2:]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


def explorer_line(dev):
    """SURVEY.md §8(f) row 2, measured beside the main path (rank 0): every
    interleaving of interval 0 of App. A.3's K_inc (lost update) at n = 6 with
    shared-access scheduling — 7 484 400 schedules — through rc_explore.  The
    start state needs no oracle: A[0] = 40, zero registers, pc 0, all running.
    Best of 3 complete calls, CUDA events on the calling stream."""
    import torch

    from paper_1308_3203_b200 import rc_explore, rc_load_program
    from workloads import kernels as K
    n = 6
    prog = rc_load_program(K.program(K.BENIGN["K_inc"]).bytecode)
    heap = torch.zeros(1 + n, dtype=torch.int32, device=dev)
    heap[0] = 40
    regs = torch.zeros((n, prog.n_regs), dtype=torch.int32, device=dev)
    pc = torch.zeros(n, dtype=torch.int32, device=dev)
    st = torch.zeros(n, dtype=torch.uint8, device=dev)
    end = 33592320  # the largest radix product of this interval: one call is complete (asserted)
    times, r = [], None
    for it in range(4):  # the first call allocates the cached buffers (untimed)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = rc_explore(prog, n, heap, regs=regs, pc=pc, status=st, sizes=[1, n], index_end=end, reduced=True)
        e1.record()
        torch.cuda.synchronize(dev)
        if it:
            times.append(e0.elapsed_time(e1))
    best = min(times)
    assert r.complete and r.n_schedules == 7484400  # 12! / 2^6 interleavings of 6 x (LD, ST)
    return {"workload": "K_inc (App. A.3) n=6, interval 0, shared-access scheduling", "schedules": r.n_schedules,
            "indices": end, "schedules_differing_from_schedule_0": r.n_differ, "ms": best,
            "schedules_per_s": r.n_schedules / (best / 1e3), "bound": "alu (issue; profiles/r01_explore_ncu_prof.txt)"}


def cpu_cores():
    return len(os.sched_getaffinity(0))


def oracle_sample(wl, n_inst, threads):
    """The oracle as it stands on a bounded sample: the first n_inst instances."""
    import oracle
    p = wl["src"]()
    ins = wl["gen"](0, n_inst, wl["n"])
    t0 = time.perf_counter()
    r = oracle.run(p.bytecode, wl["n"], ins, threads=threads, want_final=False)
    dt = time.perf_counter() - t0
    return r.stats["checked_accesses"], dt


def instances_of(wl, scaling, world):
    """(total instances of the job, instances per rank) for a workload."""
    total = wl["total"] * world if scaling == "weak" else wl["total"]
    return total, total // world


def run_reference(args, wl):
    """--impl reference: the CPU oracle timed on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = cpu_cores()
    sample = min(wl["total"], cores)
    for _ in range(args.warmup):
        oracle_sample(wl, sample, cores)
    acc = 0
    tot = 0.0
    for _ in range(args.steps):
        a, dt = oracle_sample(wl, sample, cores)
        acc += a
        tot += dt
    v = acc / tot / 1e9
    total, _ = instances_of(wl, args.scaling, args.gpus)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "int32",
            "data": "synthetic",
            "config": {"workload": wl["name"], "work_items": wl["n"], "instances_total": total,
                       "sample_instances_per_step": sample},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"first {sample} instances of the workload per step (oracle/oracle.c, "
                                       f"{cores} threads over instances)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _sum_profiles(acc, prof):
    if prof is None:
        return acc
    if acc is None:
        return prof
    for k, v in prof.items():
        if isinstance(v, dict):
            for kk in v:
                acc[k][kk] += v[kk]
        elif k != "sample_every":
            acc[k] += v
    return acc


class Job:
    """One workload's shard on this rank: program, inputs resident in HBM, the
    per-step call (rc_run + the N>1 gather)."""

    def __init__(self, wl, lo, hi, dev, local, stream, world, cdev, args):
        from paper_1308_3203_b200 import rc_load_program
        self.wl, self.lo, self.hi, self.n = wl, lo, hi, wl["n"]
        self.dev, self.local, self.stream, self.world, self.cdev, self.args = dev, local, stream, world, cdev, args
        self.prog = rc_load_program(wl["src"]().bytecode)
        self.host = wl["gen"](lo, hi, self.n)
        import torch
        self.arrays = [torch.from_numpy(x).to(dev) for x in self.host]

    def step(self, profile=False, arrs=None):
        from paper_1308_3203_b200 import rc_run
        from paper_1308_3203_b200.gather import gather_reports
        a = self.args
        r = rc_run(self.prog, self.n, arrs if arrs is not None else self.arrays, instance_offset=self.lo,
                   want_final=False, profile=profile, device=self.local, stream=self.stream,
                   keep_all_reads=a.keep_all_reads, classify_rw=a.classify_rw, prepass=getattr(a, "prepass", False))
        if self.world > 1:
            reps, st = gather_reports(r.reports, r.stats, device=self.cdev)
        else:
            reps, st = r.reports, r.stats
        return r, reps, st

    def timed(self, steps, warmup, profile=False, flush=None):
        """W untimed steps, then K timed steps (CUDA events on the launch
        stream; with `flush` an untimed L2 flush before every timed step).
        Returns (ms per step, max over ranks; accesses per step, whole job;
        instructions per step; reports per step; summed profile)."""
        import torch
        import torch.distributed as dist
        for _ in range(warmup):
            self.step()
        if self.world > 1:
            dist.barrier()
        torch.cuda.synchronize(self.dev)
        prof = None
        acc = ins = nrep = 0
        ms = 0.0
        evs = []
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        if flush is None:
            e0.record(self.stream)
        for _ in range(steps):
            if flush is not None:
                flush()
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(self.stream)
            r, reps, st = self.step(profile=profile)
            if flush is not None:
                a1.record(self.stream)
                evs.append((a0, a1))
            acc += st["checked_accesses"]
            ins += st["instructions"]
            nrep = len(reps)
            prof = _sum_profiles(prof, r.profile)
        if flush is None:
            e1.record(self.stream)
        torch.cuda.synchronize(self.dev)
        ms = sum(a.elapsed_time(b) for a, b in evs) if flush is not None else e0.elapsed_time(e1)
        if self.world > 1:
            t = torch.tensor([ms], device=self.cdev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        return ms / steps, acc // steps, ins // steps, nrep, prof


def secondary_line(key, args, world, rank, dev, local, stream, cdev, scaling, steps, warmup, flush=None):
    """A second configuration measured beside the main line (north_star covers
    stencils AND reductions): value, ms per step, accesses per step."""
    from paper_1308_3203_b200.gather import shard
    wl = WORKLOADS[key]
    total = wl["total"] * world if scaling == "weak" else wl["total"]
    if scaling == "per_gpu_share":  # BASELINE's 8-GPU configuration: every GPU its 1/8
        total = wl["total"] // 8 * world
    lo, hi = shard(total, rank, world)
    job = Job(wl, lo, hi, dev, local, stream, world, cdev, args)
    ms, acc, ins, nrep, _ = job.timed(steps, warmup, flush=flush)
    out = {"workload": wl["name"], "instances_total": total, "instances_per_gpu": hi - lo, "scaling": scaling,
           "value": acc / (ms / 1000) / 1e9, "unit": UNIT, "ms_per_step": ms, "steps": steps, "warmup": warmup,
           "checked_accesses_per_step": acc, "reports_per_step": nrep,
           "l2": "flushed (256 MB write) before every timed step" if flush else "inputs >> 126 MB L2"}
    del job
    return out


def prepass_line(args, world, rank, dev, local, stream, cdev):
    """SURVEY.md §8(f) row 4 measured beside the main line: the symbolic
    pre-pass (rc_prove, host) on config 5's shape, and the same workload run
    with RC_OPT_PREPASS — proved conflict-free, its intervals run in
    direct-commit mode without the grouping / detect kernels.  Not the
    headline: the main line measures the concrete checker."""
    import copy

    from paper_1308_3203_b200 import rc_load_program, rc_prove
    from paper_1308_3203_b200.gather import shard
    wl = WORKLOADS["cfg5"]
    prog = rc_load_program(wl["src"]().bytecode)
    sizes = [x.shape[1] for x in wl["gen"](0, 1, wl["n"])]
    t0 = time.perf_counter()
    pr = rc_prove(prog, wl["n"], sizes)
    prove_ms = (time.perf_counter() - t0) * 1e3
    a2 = copy.copy(args)
    a2.prepass = True
    total = wl["total"]
    lo, hi = shard(total, rank, world)
    job = Job(wl, lo, hi, dev, local, stream, world, cdev, a2)
    ms, acc, ins, nrep, _ = job.timed(3, 3)
    del job
    return {"workload": wl["name"], "verdict": pr.verdict, "intervals_proved": pr.intervals,
            "prove_ms": prove_ms, "prover_work": pr.work, "value": acc / (ms / 1000) / 1e9, "unit": UNIT,
            "ms_per_step": ms, "steps": 3, "warmup": 3, "reports_per_step": nrep,
            "what": "rc_run with RC_OPT_PREPASS: the symbolic NoRace pre-pass (host, cached per shape) proved the "
                    "run conflict-free, so intervals commit directly and skip the grouping / detect kernels"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg5", choices=list(WORKLOADS))
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="strong (default): the BASELINE configuration's instances split over the ranks; "
                         "weak: every rank runs the whole configuration")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--no-explorer", action="store_true", help="skip the rc_explore line (SURVEY §8(f) row 2)")
    ap.add_argument("--no-secondary", action="store_true", help="skip the config-3 / config-4 lines")
    ap.add_argument("--instances", type=int, default=0, help="override the configuration's instances (debug)")
    ap.add_argument("--classify-rw", action="store_true",
                    help="RW value classification (RC_OPT_CLASSIFY_RW, SURVEY §8(f) row 1)")
    ap.add_argument("--keep-all-reads", action="store_true",
                    help="RC_OPT_KEEP_ALL_READS: sort every read record (no write-set pruning)")
    args = ap.parse_args()
    wl = dict(WORKLOADS[args.workload])
    if args.instances:
        wl["total"] = args.instances
    if args.impl == "reference":
        return run_reference(args, wl)

    import torch
    import torch.distributed as dist

    from paper_1308_3203_b200.gather import shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE {world}"
    # (RC_BENCH_BACKEND=gloo: test hook that runs the N>1 path on one GPU —
    # ranks share device 0 — when no multi-GPU box is at hand)
    backend = os.environ.get("RC_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend == "gloo" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cdev = dev if backend == "nccl" else torch.device("cpu")  # where collectives' tensors live
    group_info = {"backend": None, "world_size": 1}
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        # the communicator's own rank count (the driver checks every rank joined)
        group_info = {"backend": dist.get_backend(), "world_size": dist.get_world_size()}
        probe = torch.ones(1, device=cdev)
        dist.all_reduce(probe)
        group_info["all_reduce_ranks"] = int(probe.item())
        if rank == 0:
            print(f"bench: process group {group_info}", file=sys.stderr, flush=True)
    total_inst, _ = instances_of(wl, args.scaling, world)
    lo, hi = shard(total_inst, rank, world)
    n = wl["n"]
    stream = torch.cuda.current_stream(dev)
    job = Job(wl, lo, hi, dev, local, stream, world, cdev, args)

    with Clocks(local) as clk:
        ms_step, acc_step, ins_step, n_reports, prof_sum = job.timed(args.steps, args.warmup,
                                                                     profile=not args.no_profile)
    # accesses already sum all ranks (gathered stats) at N>1
    value = acc_step / (ms_step / 1000) / 1e9

    # ---- end to end through the C ABI with HOST buffers (RC_OPT_HOST_IO)
    e2e = None
    if not args.no_e2e:
        pinned = [torch.from_numpy(x).pin_memory() for x in job.host]
        h2d = sum(x.numel() * 4 for x in pinned)
        job.step(arrs=pinned)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        acc2 = 0
        d2h = 0
        a0.record(stream)
        for _ in range(args.e2e_steps):
            r, reps, st = job.step(arrs=pinned)
            acc2 += st["checked_accesses"]
            d2h = len(r.reports) * 32 + 13 * 8
        a1.record(stream)
        torch.cuda.synchronize(dev)
        ems = a0.elapsed_time(a1)
        if world > 1:
            t = torch.tensor([ems], device=cdev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": acc2 / args.e2e_steps / (ems / args.e2e_steps / 1000) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
               "ms_per_step": ems / args.e2e_steps,
               "what": "rc_run with pinned host arrays (RC_OPT_HOST_IO): the H2D copy of every input inside the "
                       "step, the reports and counters back; final heaps not requested (optional in the ABI)"}
        del pinned
    del job
    torch.cuda.empty_cache()

    # ---- secondary configurations (every rank takes part in their gathers)
    secondary = None
    if not args.no_secondary and args.workload == "cfg5" and not args.instances:
        secondary = {}
        flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

        def flush():
            flush_buf.fill_(1)
        for key, scaling, steps, flush_fn in (("cfg4", "per_gpu_share", 3, None), ("cfg3", "strong", 5, flush)):
            try:
                secondary[key] = secondary_line(key, args, world, rank, dev, local, stream, cdev, scaling,
                                                steps, 3, flush=flush_fn)
            except Exception as ex:  # noqa: BLE001 — a side measurement never costs the main line
                secondary[key] = {"error": f"{type(ex).__name__}: {ex}"}
        del flush_buf
        try:  # §8(f) row 4 (every rank takes part, as in the main line)
            secondary["prepass"] = prepass_line(args, world, rank, dev, local, stream, cdev)
        except Exception as ex:  # noqa: BLE001
            secondary["prepass"] = {"error": f"{type(ex).__name__}: {ex}"}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    PER_INTERVAL = ("interp", "filter", "hist", "sort", "detect", "boundary")
    clocks = clk.summary()
    clk_mhz = clocks.get("sm_mhz")  # median SM clock during the timed steps
    n_sms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak, peak_src = peaks()
    roofline = roofline_sort = roofline_detect = None
    kernels = None
    gpu_launches = None
    if prof_sum:
        every = max(1, int(prof_sum.get("sample_every", 1)))
        s = prof_sum["sort"]
        achieved = s["alg_bytes"] / (s["ms"] / 1e3) / 1e9 if s["ms"] > 0 else None
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        tr = {}
        if os.path.exists(tpath):
            with open(tpath) as f:
                tr = json.load(f)
        lsd = bool(os.environ.get("RC_SORT_LSD"))
        sort_k = "onesweep_kernel" if lsd else "bucket_scatter_kernel"
        det_k = "detect_kernel" if lsd else "bucket_detect_kernel"
        roofline_sort = {"kernel": ("onesweep_kernel (K3, one LSD digit pass)" if lsd else
                                    "bucket_scatter_kernel (K3, MSD scatter of the kept records into 4096-cell buckets)"),
                         "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if achieved else None,
                         "traffic": tr.get(sort_k, {}).get("dram_bytes_per_launch"),
                         "alg_bytes_per_launch": s["alg_bytes"] / max(1, s["launches"]),
                         "alg_bytes_per_record": 16, "launches_sampled": s["launches"],
                         "sampling": f"CUDA events around every {every}th interval's kernels of the timed steps",
                         "peak_source": peak_src,
                         "library_sort_same_keys": cub_baseline()}
        if not s["launches"]:  # (K1c placed every write record; the workload logs no read record)
            roofline_sort = {"kernel": roofline_sort["kernel"], "launched": False,
                             "note": "not launched: K1c writes the write records straight into their bucket regions "
                                     "and no read record of this workload survives the static write-set elision"}
        # the detect kernel (K4+K5): every grouped record read, one value
        # gathered and one cell committed per write record
        dd = prof_sum["detect"]
        dach = dd["alg_bytes"] / (dd["ms"] / 1e3) / 1e9 if dd["ms"] > 0 else None
        roofline_detect = {"kernel": (det_k + " (K4+K5, " +
                                      ("segmented detect + commit, A4 tail)" if lsd else
                                       "per-bucket counting sort in shared memory + segmented detect + commit, A4 tail)")),
                           "bound": "hbm", "achieved": dach, "peak": peak, "unit": "GB/s",
                           "frac": dach / peak if dach else None,
                           "traffic": tr.get(det_k, {}).get("dram_bytes_per_launch"),
                           "alg_bytes_per_launch": dd["alg_bytes"] / max(1, dd["launches"]),
                           "alg_bytes": "8 per grouped record + 8 per write record"}
        # the interpreter (K1), the dominant kernel (largest share of the
        # step): issue-bound (ALU/LSU pipes, no contraction).  Achieved = ncu's
        # warp instructions of one launch / (live average launch duration x SM
        # clock x SMs); peak = 4 warp instructions per cycle per SM (4 SMSPs,
        # 1 issue each).
        di = prof_sum["interp"]
        ti = tr.get("interp_kernel", {})
        ipc = None
        if di["ms"] > 0 and di["launches"] and ti.get("warp_instructions_per_launch") and clk_mhz:
            avg_s = di["ms"] / di["launches"] / 1e3
            ipc = ti["warp_instructions_per_launch"] / (avg_s * clk_mhz * 1e6 * n_sms)
        roofline = {"kernel": "interp_kernel (K1, bytecode interpreter; the dominant kernel)", "bound": "alu",
                    "achieved": ipc, "peak": 4.0, "unit": "warp-instr/cycle/SM",
                    "frac": ipc / 4.0 if ipc else None,
                    "ncu_ipc_per_sm": ti.get("ipc_per_sm"),
                    "peak_source": "B200: 4 SMSPs per SM, one warp instruction issued per SMSP per cycle",
                    "traffic": ti.get("dram_bytes_per_launch"),
                    "traffic_note": "DRAM bytes of one captured launch (heap loads, lane state, staged records)"}
        if prof_sum.get("k1c"):
            # K1c, the interval kernel compiled for the program (the dominant
            # kernel): no fetch / decode left, bound by the bytes it moves —
            # status + pc in and out, the carried registers, 4 B per heap load,
            # the log; achieved = those algorithmic bytes of the
            # sampled launches / their CUDA-event time
            tk = tr.get("rc_k1c", {})
            kach = di["alg_bytes"] / (di["ms"] / 1e3) / 1e9 if di["ms"] > 0 and di["alg_bytes"] else None
            kipc = None
            if di["ms"] > 0 and di["launches"] and tk.get("warp_instructions_per_launch") and clk_mhz:
                kipc = tk["warp_instructions_per_launch"] / (di["ms"] / di["launches"] / 1e3 * clk_mhz * 1e6 * n_sms)
            roofline = {"kernel": "rc_k1c (K1c: the interval kernel compiled for the program with NVRTC; the "
                                  "dominant kernel)",
                        "bound": "hbm", "achieved": kach, "peak": peak, "unit": "GB/s",
                        "frac": kach / peak if kach else None, "peak_source": peak_src,
                        "traffic": tk.get("dram_bytes_per_launch"),
                        "alg_bytes_per_launch": di["alg_bytes"] / max(1, di["launches"]),
                        "alg_bytes": "10 per lane (status, pc in/out) + 8 per carried register and lane + 4 per heap "
                                     "load + 8 per logged read + 12 per write record (record, final value)",
                        "launches_sampled": di["launches"],
                        "issue": {"achieved": kipc, "peak": 4.0, "unit": "warp-instr/cycle/SM",
                                  "frac": kipc / 4.0 if kipc else None, "ncu_ipc_per_sm": tk.get("ipc_per_sm")}}
        kernels = {"sample_every": every}
        for c in ("interp", "filter", "hist", "sort", "detect", "boundary", "finalize", "copy"):
            d = prof_sum[c]
            k = every if c in PER_INTERVAL else 1  # sampled classes: per-step totals are estimates
            kernels[c] = {"launches_per_step": k * d["launches"] / args.steps, "ms_per_step": k * d["ms"] / args.steps,
                          "share": k * d["ms"] / prof_sum["total_ms"] if prof_sum["total_ms"] else None,
                          "alg_GBps": d["alg_bytes"] / (d["ms"] / 1e3) / 1e9 if d["ms"] > 0 and d["alg_bytes"] else None}
        kernels["total_ms_per_step"] = prof_sum["total_ms"] / args.steps
        gpu_launches = prof_sum["kernel_launches"]

    cpu = None
    if not args.no_cpu_baseline:  # rank 0 (the others wait at the final barrier)
        cores = cpu_cores()
        sample = min(total_inst, 2 * cores)
        acc, dt = oracle_sample(wl, sample, cores)
        cpu = {"value": acc / dt / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"first {sample} instances of the workload ({n} work-items each), "
                         f"{cores} threads over instances, {dt:.1f} s (rank 0)"}

    explorer = None
    if not args.no_explorer:
        try:  # a side measurement: never costs the main line
            explorer = explorer_line(dev)
        except Exception as ex:  # noqa: BLE001
            explorer = {"error": f"{type(ex).__name__}: {ex}"}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": wl["name"], "work_items": n, "instances_total": total_inst,
                       "instances_per_gpu": hi - lo, "write_set_filter": not args.keep_all_reads,
                       "classify_rw": args.classify_rw, "final_heaps": False,
                       "parallelism": f"dp{world} (contiguous instance shards, NCCL gather of reports)",
                       "process_group": group_info,
                       "l2": "inputs 4.3 GB in all >> 126 MB L2 (no flush needed)",
                       "checked_accesses_per_step": acc_step, "reports_per_step": n_reports},
            "roofline": roofline, "roofline_sort": roofline_sort, "roofline_detect": roofline_detect,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": gpu_launches,
            "interpreter": {"bytecode_instr_per_s": ins_step / (ms_step / 1000),
                            "bytecode_instr_per_step": ins_step,
                            "executed_by": "K1c (the interval kernel compiled for the program)" if
                            (prof_sum or {}).get("k1c") else "K1 (the bytecode interpreter)"},
            "clocks": clocks, "kernels": kernels, "secondary": secondary, "explorer": explorer}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
