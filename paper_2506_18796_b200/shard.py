"""Multi-GPU scenario sharding for one process per GPU.

Scenarios are fully independent, so a sweep is split into shards, one per
rank, with the same assignment the single-process multi-device entry
(cace_replay_batch_multi) uses: every (capacity, trace) group is cut into
warps of 32 scenarios spread evenly over the shards (cace_shard_scenarios),
so every rank replays the same mix and no cost model is needed.  Every rank
holds a replica of the traces and catalog, replays its shard with no
data-path communication, and the fixed-size per-scenario summaries (112 B
each) are all-gathered once at the end -- the only collective (NCCL over
NVLink/NVSwitch on the GPU box; gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np

from ._native import SUMMARY_DTYPE


def shard_indices(sc: np.ndarray, n_models: int, world: int) -> list[np.ndarray]:
    """Scenario indices of each rank's shard (ascending)."""
    from .api import shard_scenarios

    of = shard_scenarios(sc, n_models, world)
    return [np.nonzero(of == r)[0] for r in range(world)]


def gather_summaries(local, parts: list[np.ndarray], group=None):
    """All-gather per-rank summary shards (torch uint8 tensors of
    len(shard) * 112 bytes, in shard order) -> the full summary array in the
    sweep's order (numpy, SUMMARY_DTYPE) on every rank.  Shards are padded to
    the largest so one collective moves everything."""
    import torch
    import torch.distributed as dist

    world = len(parts)
    width = SUMMARY_DTYPE.itemsize
    max_rows = max(len(p) for p in parts)
    pad = torch.zeros(max(max_rows, 1) * width, dtype=torch.uint8, device=local.device)
    pad[: local.numel()].copy_(local)
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    n = sum(len(p) for p in parts)
    full = np.zeros(n, SUMMARY_DTYPE)
    for r in range(world):
        rows = len(parts[r])
        full[parts[r]] = outs[r][: rows * width].cpu().numpy().view(SUMMARY_DTYPE)
    return full
