"""Multi-GPU scenario sharding.

Scenarios are fully independent, so a sweep is split into contiguous,
cost-balanced shards, one per rank (one process per GPU).  Every rank holds
a replica of the traces and catalog, replays its shard with no data-path
communication, and the fixed-size per-scenario summaries (112 B each) are
all-gathered once at the end — the only collective (NCCL over
NVLink/NVSwitch on the GPU box; gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np

from ._native import SUMMARY_DTYPE


def scenario_cost(sc: np.ndarray) -> np.ndarray:
    """Relative replay cost of each scenario: the per-decision work grows with
    the lookahead window (rank scan) and with capacity (slot scans)."""
    w = np.maximum(sc["window_length"].astype(np.float64), 1.0)
    c = sc["num_accelerators"].astype(np.float64) * np.maximum(sc["models_per_accelerator"], 1)
    return 1.0 + np.log2(w) / 8.0 + c / 8.0


def shard_bounds(sc: np.ndarray, world: int) -> list[int]:
    """Contiguous [b_r, b_{r+1}) bounds with ~equal summed cost."""
    cum = np.concatenate([[0.0], np.cumsum(scenario_cost(sc))])
    bounds = [0]
    for r in range(1, world):
        bounds.append(int(np.searchsorted(cum, cum[-1] * r / world)))
    bounds.append(len(sc))
    return bounds


def gather_summaries(local, bounds: list[int], group=None):
    """All-gather per-rank summary shards (torch uint8 tensors of
    len(shard) * 112 bytes) -> full summary array (numpy, SUMMARY_DTYPE) on
    every rank.  Shards are padded to the largest so one collective moves
    everything."""
    import torch
    import torch.distributed as dist

    world = len(bounds) - 1
    width = SUMMARY_DTYPE.itemsize
    max_rows = max(bounds[r + 1] - bounds[r] for r in range(world))
    pad = torch.zeros(max_rows * width, dtype=torch.uint8, device=local.device)
    pad[: local.numel()].copy_(local)
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    parts = []
    for r in range(world):
        rows = bounds[r + 1] - bounds[r]
        parts.append(outs[r][: rows * width].cpu().numpy())
    return np.concatenate(parts).view(SUMMARY_DTYPE)
