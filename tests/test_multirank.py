"""N > 1 path on CPU: world_size-2 gloo run of the replica timing reduction
used by bench.py (max over ranks, whole-job throughput), and a replica solve
on each rank with the CPU oracle to show ranks are independent."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1903_10977_b200.replicas import job_throughput
    ms, value = job_throughput(10.0 * (rank + 1), 1000, world, dist)
    # each replica solves its own copy (here with the oracle on CPU)
    import oracle_ffi as orc
    from paper_1903_10977_b200 import build_case, configs
    case = build_case(configs.c1(threads=1))
    st, x, res, it, _ = orc.pcg(case.levels_c(), case.b, tol=1e-8)
    out[rank] = (ms, value, st, it)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_replica_timing_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert len(out) == 2
    for r in range(world):
        ms, value, st, it = out[r]
        assert ms == 20.0                      # max over ranks
        assert value == pytest.approx(1000 * 2 / 0.020)
        assert st == 0 and it == out[0][3]     # identical replicas
