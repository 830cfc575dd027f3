"""Multi-GPU segment model (the paper's per-machine segment
indexes).

One process per GPU, torch.distributed for the plumbing.  A single HNSW build
does not shard (every insertion walks data-dependent paths over the whole
graph, reverse edges hit arbitrary rows), so N GPUs build N independent
segment indexes over disjoint row ranges with no collective on the build path
except one broadcast of the trained coder.  A query runs on every segment;
the per-segment top-k lists (global ids, distances) are all-gathered and
merged by (distance, global id) — the reference's result order (fa_pair_cmp,
_simd.h:237-243) — into the global top-k.
"""

from __future__ import annotations

import numpy as np

from .flash import FlashModel, FlashProvider


def segment_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [lo, hi) of segment `rank` of `world` (sizes differ by at most 1)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def broadcast_model(model: FlashModel | None, src: int = 0, group=None) -> FlashModel:
    """The coder trained on rank `src`, on every rank (one broadcast)."""
    import torch.distributed as dist

    box = [FlashProvider(model).state_dict() if dist.get_rank(group) == src else None]
    dist.broadcast_object_list(box, src=src, group=group)
    return FlashProvider.from_state(box[0]).model


def merge_topk(ids, dists, base: int, k: int, group=None):
    """Global top-k from per-segment results.

    ids (nq, k) int64 local ids, -1 padded; dists (nq, k) float64, +inf padded
    (search_batch's outputs); `base` = this segment's first global row.  The
    tensors live where the process group's backend wants them (CUDA for NCCL,
    CPU for gloo).  Returns (ids, dists) with global ids, on every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    gid = torch.where(ids >= 0, ids + base, torch.full_like(ids, -1))
    all_ids = [torch.empty_like(gid) for _ in range(world)]
    all_d = [torch.empty_like(dists) for _ in range(world)]
    dist.all_gather(all_ids, gid, group=group)
    dist.all_gather(all_d, dists, group=group)
    return merge_lists(torch.cat(all_ids, 1), torch.cat(all_d, 1), k)


def merge_lists(ids, dists, k: int):
    """First k of each row by (distance, id); padding (-1, +inf) sorts last."""
    import torch

    key_id = torch.where(ids >= 0, ids, torch.full_like(ids, torch.iinfo(ids.dtype).max))
    o = torch.argsort(key_id, dim=1, stable=True)
    ids, dists, key_id = ids.gather(1, o), dists.gather(1, o), key_id.gather(1, o)
    o = torch.argsort(dists, dim=1, stable=True)
    return ids.gather(1, o)[:, :k], dists.gather(1, o)[:, :k]


def merge_lists_np(ids: np.ndarray, dists: np.ndarray, k: int):
    """numpy twin of merge_lists (single process, for checks)."""
    key_id = np.where(ids >= 0, ids, np.iinfo(ids.dtype).max)
    out_i = np.empty((ids.shape[0], k), ids.dtype)
    out_d = np.empty((ids.shape[0], k), dists.dtype)
    for r in range(ids.shape[0]):
        o = np.lexsort((key_id[r], dists[r]))[:k]
        out_i[r], out_d[r] = ids[r, o], dists[r, o]
    return out_i, out_d
