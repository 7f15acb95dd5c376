"""N>1 path through the real product: world_size-2
processes each run rc_run (librc.so, the CUDA path) on their contiguous
instance shard (instance_offset = shard start) and gather_reports joins the
shards; the result must equal one rc_run over all instances byte for byte —
reports in canonical order and every counter.

* gloo: both ranks share cuda:0 (the collectives move CPU tensors), so this
  runs on the one-GPU test box;
* nccl: one GPU per rank, collectives on the GPUs; skipped below 2 GPUs.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from workloads import inputs as I  # noqa: E402
from workloads import kernels as K  # noqa: E402

CASES = {
    "tree_off_by_one": (lambda: K.program(K.TREE_OFF_BY_ONE), 64, lambda lo, hi: I.cfg3_inputs(lo, hi, 64), 11),
    "cfg4": (lambda: K.random_stencil_kernel(3), 300, lambda lo, hi: _cfg4(lo, hi), 6),
    "benign_Btid": (lambda: K.program(K.BENIGN["K_Btid"]), 256, lambda lo, hi: I.cfg2_inputs(lo, hi, 256), 9),
}


def _cfg4(lo, hi):
    ins = I.cfg4_inputs(lo, hi, 300)
    ins[3][:, 30:70] += 1  # dense perturbation: input-dependent races in every instance
    return ins


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, backend, case, q):
    import torch
    import torch.distributed as dist

    from paper_1308_3203_b200 import rc_load_program, rc_run
    from paper_1308_3203_b200.gather import gather_reports, shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev_i = rank if backend == "nccl" else 0
    torch.cuda.set_device(dev_i)
    dev = torch.device("cuda", dev_i)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    src, n, gen, n_inst = CASES[case]
    lo, hi = shard(n_inst, rank, world)
    prog = rc_load_program(src().bytecode)
    r = rc_run(prog, n, [torch.from_numpy(x).to(dev) for x in gen(lo, hi)], instance_offset=lo, device=dev_i,
               want_final=False)
    reps, st = gather_reports(r.reports, r.stats, device=dev if backend == "nccl" else None)
    if rank == 0:
        q.put((reps.tobytes(), st, dist.get_world_size()))
    dist.destroy_process_group()


def _run(backend, case):
    import torch.multiprocessing as mp

    from paper_1308_3203_b200 import rc_load_program, rc_run
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, backend, case, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got, st, ws = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    assert ws == 2
    src, n, gen, n_inst = CASES[case]
    ref = rc_run(rc_load_program(src().bytecode), n, [torch.from_numpy(x).cuda() for x in gen(0, n_inst)],
                 want_final=False)
    assert len(ref.reports) > 0
    assert got == ref.reports.tobytes()
    for k in ("checked_accesses", "loads", "stores", "instructions", "intervals_max", "lanes_final"):
        assert st[k] == ref.stats[k], k


@pytest.mark.parametrize("case", list(CASES))
def test_shards_gather_gloo(case):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _run("gloo", case)


@pytest.mark.parametrize("case", list(CASES))
def test_shards_gather_nccl(case):
    if torch.cuda.device_count() < 2:
        pytest.skip("NCCL gather needs 2 GPUs")
    _run("nccl", case)


def test_bench_two_ranks_strong_scaling():
    """bench.py at N=2 (two ranks sharing cuda:0 over gloo, the test hook
    RC_BENCH_BACKEND=gloo): strong scaling of config 5's instances — the job
    still checks 512 instances (a reduced instance count keeps it short)."""
    import json
    import subprocess
    import sys
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RC_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"), "--gpus", "2",
           "--steps", "2", "--warmup", "1", "--instances", "8", "--no-e2e", "--no-explorer", "--no-secondary"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["instances_total"] == 8 and line["config"]["instances_per_gpu"] == 4
    assert line["config"]["process_group"]["world_size"] == 2
    assert line["config"]["checked_accesses_per_step"] == 24 * (1 << 20) * 8
    assert line["cpu_baseline"] is not None
