"""Query-time search and recall (mirrors flashann/evaluation.py:26-98).

search_batch runs the device search (K8: descent, layer-0 search of width
ef, optional exact fp32 rerank with (d, id) ordering) over a GPU-resident
GraphIndex.  recall = |G intersect S| / k (evaluation.py:23).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check
from .errors import ConfigError

RECALL_FORMULA = "recall = |G intersect S| / k"


@dataclass
class SearchParams:
    ef: int
    k: int = 1
    rerank_depth: int = 0

    def __post_init__(self):
        if self.k < 1 or self.ef < self.k:
            raise ConfigError(f"need 1 <= k <= ef, got k={self.k} ef={self.ef}")
        if self.rerank_depth and self.rerank_depth < self.k:
            raise ConfigError("rerank_depth must be >= k when reranking is on")


def search_batch_dev(g, provider, queries_dev, params: SearchParams, stream=None):
    """Device-resident search: (ids (nq,k) int64, dists (nq,k) f64) as device
    tensors, plus counters."""
    import torch

    lib = _lib.load()
    nq = queries_dev.shape[0]
    qp = provider.query_aux_dev(queries_dev)
    ids = torch.empty((nq, params.k), dtype=torch.int64, device="cuda")
    ds = torch.empty((nq, params.k), dtype=torch.float64, device="cuda")
    ctr = np.zeros(4, np.int64)
    check(lib.fa_index_search(g.handle, queries_dev.data_ptr(), qp.data_ptr(), nq, params.ef,
                              params.k, params.rerank_depth, g.entry_point, g.max_layer,
                              ids.data_ptr(), ds.data_ptr(), _lib.ptr(ctr), stream))
    return ids, ds, {"dist_comps": int(ctr[0]), "sym_comps": int(ctr[1]),
                     "kernel_calls": int(ctr[2]), "visited": int(ctr[3])}


def search_batch(g, provider, queries, params: SearchParams, threads: int = 1,
                 kernel: str | None = None, core_impl=None):
    """Top-k ids and squared distances for each query row."""
    from .pca import as_device_f32

    q = np.ascontiguousarray(np.atleast_2d(queries), dtype=np.float32)
    if q.shape[1] != g.dim:
        raise ConfigError(f"query dimension {q.shape[1]} != index dimension {g.dim}")
    if g.entry_point < 0:
        raise ConfigError("cannot search an empty graph")
    if core_impl is not None:
        return core_impl.search_batch(
            provider.kind_id, provider.core_arrays(), g.levels, g.base_blocks, g.upper_offsets,
            g.upper_blocks, g.params.C, g.params.R, g.entry_point, g.max_layer, q,
            provider.query_aux(q), params.ef, params.k, params.rerank_depth, threads=threads,
            kernel=0)
    if g.handle is None:
        raise ConfigError("graph has no device index; pass core_impl for host arrays")
    ids, ds, ctr = search_batch_dev(g, provider, as_device_f32(q), params)
    return ids.cpu().numpy(), ds.cpu().numpy(), ctr


def search(g, provider, query, params: SearchParams, kernel=None, core_impl=None):
    ids, dists, _ = search_batch(g, provider, np.atleast_2d(query), params, core_impl=core_impl)
    return [(int(i), float(d)) for i, d in zip(ids[0], dists[0]) if i >= 0]


def recall_at_k(result_ids: np.ndarray, gt) -> float:
    k = gt.k
    hits = 0
    for row, truth in zip(result_ids, gt.ids):
        hits += len(set(int(i) for i in row[:k] if i >= 0) & set(int(t) for t in truth[:k]))
    return hits / (len(gt.ids) * k)
