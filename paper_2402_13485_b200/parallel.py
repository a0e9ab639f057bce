"""Multi-GPU plumbing: one model replica per rank, sequences sharded in
contiguous ranges, and the per-step exchange of acceptance records.

The only data-path collective is `all_gather_records`: each rank contributes
its [B_r, D] int8 acceptance records (1-based rank of the realized token in
the head's draft list, -1 miss, 0 unknown depth) and receives the global
[sum B_r, D] table in rank order, which is global sequence order.  Every
rank then replays the fp64 statistics update in that order on its own device
(propd_stats_replay_select), so all replicas hold bit-identical P and plan
the same tree — the reference's single-process update order
(engine.py:257-288, acceptance.py:96-113).  Summing float hit counts with an
all-reduce would not be bit-exact because the EMA is order-dependent.

Works over NCCL (CUDA tensors) and gloo (CPU tensors, used by the CPU tests).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def _dev(group):
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else torch.device("cpu")


def all_gather_records(local: torch.Tensor, group=None) -> torch.Tensor:
    """Concatenate every rank's [B_r, D] int8 records in rank order."""
    dev = _dev(group)
    world = dist.get_world_size(group)
    D = local.shape[1]
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    cap = max(max(sizes), 1)
    buf = torch.zeros(cap, D, dtype=torch.int8, device=dev)
    if local.shape[0]:
        buf[: local.shape[0]] = local.to(dev)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    out = torch.cat([p[:s] for p, s in zip(parts, sizes)], dim=0)
    return out.to(local.device)


def all_reduce_scalars(vals, op: str, group=None):
    """Sum/max of a few python scalars across ranks (ints stay ints)."""
    dev = _dev(group)
    is_int = [isinstance(v, (int,)) and not isinstance(v, bool) for v in vals]
    t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX, group=group)
    return [int(round(x)) if i else float(x) for x, i in zip(t.tolist(), is_int)]


def all_gather_ints(vals, group=None) -> list:
    """Concatenation of every rank's int list, in rank order."""
    dev = _dev(group)
    local = torch.tensor(list(vals), dtype=torch.int64, device=dev).view(-1, 1)
    recs = all_gather_records_int64(local, group)
    return [int(v) for v in recs.view(-1).tolist()]


def all_gather_records_int64(local: torch.Tensor, group=None) -> torch.Tensor:
    dev = _dev(group)
    world = dist.get_world_size(group)
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    cap = max(max(sizes), 1)
    buf = torch.zeros(cap, local.shape[1], dtype=torch.int64, device=dev)
    if local.shape[0]:
        buf[: local.shape[0]] = local.to(dev)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)], dim=0)


def all_gather_objects(obj, group=None) -> list:
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out
