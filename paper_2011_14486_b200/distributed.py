"""Multi-GPU helpers: one process per GPU, torch.distributed
for the plumbing.

Scoring shards with no data-path collective beyond gathering results:
`predict_states_sharded` gives rank r the contiguous slice r of the global
state list and all-gathers the V values so every rank holds the full vector
(in the original order).  `global_argmin` reduces a per-rank candidate slice
to the reference's argmin - lowest value, ties to the lowest global index
(search.py:110) - exactly: a MIN all-reduce of the f64 values, then a MIN
all-reduce of the indices that hold that value (V > 0, so f64 order is the
int64 order of the bits and no precision is lost).
"""

from __future__ import annotations

import numpy as np


def shard_range(n: int, rank: int, world: int) -> tuple:
    """Contiguous [lo, hi) of n items for `rank` (sizes differ by <= 1)."""
    return (n * rank) // world, (n * (rank + 1)) // world


def predict_states_sharded(params, states, dist, scorer=None, **kw) -> np.ndarray:
    """V for all `states` on every rank; each rank scores only its slice."""
    import torch
    if scorer is None:
        from .value_model import predict_states as scorer
    world, rank = dist.get_world_size(), dist.get_rank()
    n = len(states)
    lo, hi = shard_range(n, rank, world)
    mine = np.asarray(scorer(params, states[lo:hi], **kw), dtype=np.float64)
    counts = [shard_range(n, r, world) for r in range(world)]
    width = max(h - l for l, h in counts)
    dev = _dev(dist)
    buf = torch.zeros(width, dtype=torch.float64, device=dev)
    buf[: hi - lo] = torch.from_numpy(mine).to(dev)
    parts = [torch.zeros(width, dtype=torch.float64, device=dev) for _ in range(world)]
    dist.all_gather(parts, buf)
    return np.concatenate([parts[r][: h - l].cpu().numpy() for r, (l, h) in enumerate(counts)])


def global_argmin(values: np.ndarray, offset: int, dist) -> tuple:
    """(min value, lowest global index holding it) over all ranks' slices;
    `offset` is this rank's first global index."""
    import torch
    dev = _dev(dist)
    values = np.asarray(values, dtype=np.float64)
    local = float(values.min()) if len(values) else float("inf")
    v = torch.tensor([local], dtype=torch.float64, device=dev)
    dist.all_reduce(v, op=dist.ReduceOp.MIN)
    best = float(v.item())
    hit = np.flatnonzero(values == best)
    idx = torch.tensor([offset + int(hit[0]) if len(hit) else np.iinfo(np.int64).max],
                       dtype=torch.int64, device=dev)
    dist.all_reduce(idx, op=dist.ReduceOp.MIN)
    return best, int(idx.item())


def _dev(dist):
    import torch
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")
