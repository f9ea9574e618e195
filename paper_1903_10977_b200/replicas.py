"""Multi-GPU execution model: replicas only.

The north star keeps one solve on one GPU; bench.py --gpus N therefore runs N
independent replicas (one process per GPU, torchrun), each solving its own
copy of the workload with no data-path collective.  The only collectives are
control-plane: a barrier around the timed region and a MAX all-reduce of the
per-rank device time, so the job throughput is N * n_dofs / max_rank(t).
"""
from __future__ import annotations


def job_time_ms(ms_local: float, dist=None, device=None) -> float:
    """MAX over ranks of a per-rank device time (torch.distributed all_reduce)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(ms_local)
    import torch
    t = torch.tensor([float(ms_local)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(ms_local: float, n_local: int, world: int, dist=None, device=None):
    """Returns (max-over-ranks ms per step, whole-job DOF-solves/s)."""
    ms = job_time_ms(ms_local, dist, device)
    return ms, n_local * world / (ms * 1e-3)
