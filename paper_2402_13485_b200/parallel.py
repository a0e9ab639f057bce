"""Multi-GPU plumbing: one model replica per rank, sequences sharded in
contiguous ranges, and ONE collective per decode step.

Each step every rank contributes a fixed-size int32 table (`step_exchange`):
a header row [active sequences on this rank, step time in µs] and one row per
active sequence:

    [acc_len, |survivors|, tokens kept after EOS/max clipping, finished,
     rank record r_1..r_D, committed tokens c_0..c_D]

where r_d is the 1-based rank of the realized token in head d's draft list
(-1 miss, 0 depth not reached; acceptance.py:53-57, engine.py:283-288) and
c_0..c_D the accepted chain + bonus (-1 padded).  One all_gather of the table
gives every rank the whole step in global sequence order (ranks own
contiguous, increasing index ranges): every rank replays the fp64 statistics
update in that order on its own device (propd_stats_replay_select), so the
replicas hold bit-identical P, plan the same tree and agree with the
single-process reference (acceptance.py:96-113 applied per sequence in batch
order, engine.py:257-288).  Batch size, mean sequence length, prune rates,
metric sums, the wall-clock maximum and the transcripts all follow from the
same table, so there is no other per-step collective and nothing is pickled.
A sum of float hit counts would not be bit-exact: the EMA is order-dependent.

Works over NCCL (CUDA tensors) and gloo (CPU tensors; the CPU tests).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

HEADER_ACTIVE, HEADER_STEP_US = 0, 1
COL_ACC, COL_SURV, COL_KEPT, COL_FIN, COL_RANKS = 0, 1, 2, 3, 4


def record_width(D: int) -> int:
    return COL_RANKS + D + D + 1


def collective_device(group):
    """Where the exchanged tensor lives: the current GPU for NCCL, host for gloo."""
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else torch.device("cpu")


def step_exchange(rows: np.ndarray, step_us: int, cap: int, group) -> torch.Tensor:
    """All-gather of every rank's [cap + 1, R] int32 step table (header row +
    up to `cap` sequence rows) -> [world, cap + 1, R] on the collective's device."""
    dev = collective_device(group)
    world = dist.get_world_size(group)
    R = rows.shape[1]
    host = np.zeros((cap + 1, R), dtype=np.int32)
    host[0, HEADER_ACTIVE] = rows.shape[0]
    host[0, HEADER_STEP_US] = step_us
    host[1: 1 + rows.shape[0]] = rows
    buf = torch.from_numpy(host).to(dev)
    out = torch.empty(world, cap + 1, R, dtype=torch.int32, device=dev)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, buf, group=group)
    else:
        dist.all_gather(list(out.unbind(0)), buf, group=group)
    return out


def global_rows(table: torch.Tensor) -> tuple:
    """(host [S, R] int32 rows of every active sequence in global order, the
    per-rank step µs, the device/host tensor of those rows)."""
    counts = table[:, 0, HEADER_ACTIVE].tolist()
    parts = [table[r, 1: 1 + n] for r, n in enumerate(counts)]
    dev_rows = torch.cat(parts, dim=0) if parts else table[:0, 0]
    return dev_rows.cpu().numpy(), table[:, 0, HEADER_STEP_US].cpu().numpy(), dev_rows


def all_gather_objects(obj, group=None) -> list:
    """Pickled gather (end-of-run use only, never on the per-step path)."""
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out
