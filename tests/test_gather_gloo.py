"""N>1 host path on CPU: world_size-2 gloo processes shard the instances
(paper_1308_3203_b200.gather.shard), each produces its shard's reports (here
from the oracle, standing in for rc_run on its GPU), and gather_reports must
reproduce exactly the single-process result — canonical order included."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from workloads import inputs as I
from workloads import kernels as K


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_inst, q):
    import torch.distributed as dist

    import oracle
    from paper_1308_3203_b200.gather import gather_reports, shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard(n_inst, rank, world)
    p = K.program(K.TREE_OFF_BY_ONE)
    ins = I.cfg3_inputs(lo, hi, 64)
    r = oracle.run(p.bytecode, 64, ins, instance_offset=lo, threads=1)
    reps = np.frombuffer(r.reports.tobytes(), dtype=_dtype()).copy()
    out, st = gather_reports(reps, r.stats)
    if rank == 0:
        q.put((out.tobytes(), st))
    dist.destroy_process_group()


def _dtype():
    from paper_1308_3203_b200.rc import REPORT_DTYPE
    return REPORT_DTYPE


@pytest.mark.parametrize("n_inst", [9, 10])
def test_gather_two_ranks(n_inst):
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_inst, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got, st = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = K.program(K.TREE_OFF_BY_ONE)
    ref = oracle.run(p.bytecode, 64, I.cfg3_inputs(0, n_inst, 64))
    assert got == ref.reports.tobytes()
    for k in ("checked_accesses", "loads", "stores", "instructions", "intervals_max", "lanes_final"):
        assert st[k] == ref.stats[k], k


def test_shard_covers():
    from paper_1308_3203_b200.gather import shard
    for n in (0, 1, 7, 512, 4096):
        for w in (1, 2, 3, 8):
            rs = [shard(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
