"""Layered graph container on the device (mirrors flashann/graph.py).

BuildParams (:24-47), the layer draws (:55-78: splitmix64 uniforms ->
floor(-ln u / ln R)) and GraphIndex (:81-134).  The GraphIndex here owns a
device-resident fa_index (SoA adjacency + flat code table); the reference's
interleaved block arrays are produced on demand by the GPU exporter
(`base_blocks` / `upper_blocks`), so a GPU-built index can be handed to the
reference's own searcher or serialiser unchanged.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib, layout
from ._lib import check
from .errors import ConfigError


@dataclass
class BuildParams:
    C: int = 1024
    R: int = 32
    seed: int = 0
    threads: int = 1

    def __post_init__(self):
        if self.R < 2:
            raise ConfigError("R must be >= 2")
        if self.R > self.C:
            raise ConfigError(f"R={self.R} must not exceed C={self.C}")
        if self.threads < 1:
            raise ConfigError("threads must be >= 1")

    @property
    def ml(self) -> float:
        return 1.0 / math.log(self.R)

    def cap(self, layer: int) -> int:
        return 2 * self.R if layer == 0 else self.R


_PHI64 = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)


def uniform_draws(n: int, seed: int) -> np.ndarray:
    """u_i in (0, 1]: a pure function of (seed, i) (graph.py:55-69)."""
    with np.errstate(over="ignore"):
        z = np.arange(1, n + 1, dtype=np.uint64) * _PHI64 + np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
        z = (z ^ (z >> np.uint64(30))) * _MIX1
        z = (z ^ (z >> np.uint64(27))) * _MIX2
        z = z ^ (z >> np.uint64(31))
    return ((z >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53


def layer_from_uniform(u: float, R: int) -> int:
    return int(math.floor(-math.log(u) / math.log(R)))


def assign_layers(n: int, seed: int, R: int) -> np.ndarray:
    if n == 0:
        return np.zeros(0, dtype=np.int32)
    return np.floor(-np.log(uniform_draws(n, seed)) * (1.0 / math.log(R))).astype(np.int32)


def upper_offsets_of(levels: np.ndarray) -> np.ndarray:
    lv = levels.astype(np.int64)
    return np.where(lv > 0, np.cumsum(lv) - lv, -1)


class GraphIndex:
    """Adjacency of a built (or in-progress) index, resident on the GPU."""

    def __init__(self, n: int, dim: int, params: BuildParams, strategy: str,
                 code_subspaces: int, levels: np.ndarray):
        self.dim = dim
        self.params = params
        self.strategy = strategy
        self.code_subspaces = code_subspaces
        self.levels = np.ascontiguousarray(levels, dtype=np.int32)
        self.base_cap = 2 * params.R
        self.upper_cap = params.R
        self.upper_offsets = upper_offsets_of(self.levels)
        self.n_upper_rows = int(self.levels.astype(np.int64).sum())
        self.entry_point = -1
        self.max_layer = -1
        self.counters: dict = {}
        self.handle = None  # fa_index*
        self._keep: list = []
        self._blocks = None

    @property
    def n(self) -> int:
        return self.levels.shape[0]

    # ---- device handle ----------------------------------------------------
    def create_device(self, provider) -> None:
        import torch

        lib = _lib.load()
        dev = provider.dev
        lv = torch.from_numpy(self.levels).cuda()
        uo = torch.from_numpy(np.ascontiguousarray(self.upper_offsets, np.int64)).cuda()
        self._keep = [lv, uo]
        d = _lib.IndexDesc()
        if provider.kind_id == 0:  # exact strategy: m = 0, fp32 L2 over the vectors
            d.n, d.m, d.R = self.n, 0, self.params.R
            d.dim = d.dproj = int(dev["vecs"].shape[1])
            d.vecs = dev["vecs"].data_ptr()
            d.levels, d.uoff = lv.data_ptr(), uo.data_ptr()
            d.n_upper_rows = self.n_upper_rows
            self._desc = d
            h = _lib.vp()
            check(lib.fa_index_create(C.byref(d), C.byref(h)))
            self.handle = h
            self._provider = provider
            return
        model = provider.model
        d.n, d.m, d.R = self.n, model.m, self.params.R
        d.dproj = int(dev["proj"].shape[1])
        d.dmax = int(model.cent.shape[2])
        d.dist_min, d.delta = float(model.dist_min), float(model.delta)
        d.proj = dev["proj"].data_ptr()
        if dev["vecs"].dtype == torch.float32:  # rerank reads fp32 vectors
            d.vecs, d.dim = dev["vecs"].data_ptr(), int(dev["vecs"].shape[1])
        d.cent, d.dims = dev["cent"].data_ptr(), dev["dims"].data_ptr()
        d.offs, d.sdt = dev["offs"].data_ptr(), dev["sdt"].data_ptr()
        d.levels, d.uoff = lv.data_ptr(), uo.data_ptr()
        d.n_upper_rows = self.n_upper_rows
        self._desc = d
        h = _lib.vp()
        check(lib.fa_index_create(C.byref(d), C.byref(h)))
        self.handle = h
        codes = dev["codes"]
        check(lib.fa_index_set_codes(h, codes.data_ptr(), codes.shape[1], None))
        self._provider = provider

    def close(self) -> None:
        if self.handle is not None:
            _lib.load(require_device=False).fa_index_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- reference-layout view ------------------------------------------
    def export_blocks(self):
        """(base_blocks, upper_blocks) in the reference layout (host)."""
        import torch

        if self._blocks is None:
            lib = _lib.load()
            m = self.code_subspaces
            sb = layout.block_stride(self.base_cap, m)
            su = layout.block_stride(self.upper_cap, m)
            db = torch.empty((self.n, sb), dtype=torch.uint8, device="cuda")
            du = torch.empty((max(self.n_upper_rows, 1), su), dtype=torch.uint8, device="cuda")
            check(lib.fa_index_export_blocks(self.handle, db.data_ptr(), sb, du.data_ptr(), su,
                                             None))
            self._blocks = (db.cpu().numpy(), du[: self.n_upper_rows].cpu().numpy())
        return self._blocks

    @property
    def base_blocks(self) -> np.ndarray:
        return self.export_blocks()[0]

    @property
    def upper_blocks(self) -> np.ndarray:
        return self.export_blocks()[1]

    def invalidate(self) -> None:
        self._blocks = None

    def vertex_level(self, v: int) -> int:
        return int(self.levels[v])

    def _row(self, v: int, layer: int):
        if layer == 0:
            return self.base_blocks, v, self.base_cap
        if layer > self.levels[v]:
            raise ConfigError(f"vertex {v} absent from layer {layer}")
        return self.upper_blocks, int(self.upper_offsets[v]) + layer - 1, self.upper_cap

    def neighbors(self, v: int, layer: int) -> np.ndarray:
        blocks, row, cap = self._row(v, layer)
        return layout.row_ids(blocks, row, cap)

    def neighbor_codes(self, v: int, layer: int) -> np.ndarray:
        blocks, row, cap = self._row(v, layer)
        return layout.row_codes(blocks, row, cap, self.code_subspaces)

    def degree_stats(self, layer: int = 0):
        blocks = self.base_blocks if layer == 0 else self.upper_blocks
        counts = blocks[:, :4].copy().view(np.int32)[:, 0]
        return float(counts.mean()), int(counts.max())

    def core_arrays(self) -> dict:
        return {"levels": self.levels, "base_blocks": self.base_blocks,
                "upper_offsets": self.upper_offsets, "upper_blocks": self.upper_blocks}


def check_invariants(graph: GraphIndex) -> list[str]:
    """Structural sweep (graph.py:137-187): caps, self loops, id range, layer
    membership, entry point on the top layer — vectorized over the rows of
    each layer (a 1M-vertex graph checks in about a second)."""
    bad: list[str] = []
    n = graph.n
    if n == 0:
        return bad
    if not 0 <= graph.entry_point < n:
        bad.append(f"entry point {graph.entry_point} out of range")
    elif graph.levels[graph.entry_point] != graph.max_layer:
        bad.append("entry point is not on the top layer")
    if graph.levels.max(initial=0) != graph.max_layer:
        bad.append("max_layer disagrees with assigned levels")
    for layer in range(graph.max_layer + 1):
        cap = graph.params.cap(layer)
        if layer == 0:
            blocks, owners = graph.base_blocks, np.arange(n)
        else:
            owners = np.flatnonzero(graph.levels >= layer)
            rows = graph.upper_offsets[owners] + layer - 1
            blocks = graph.upper_blocks[rows] if len(rows) else graph.upper_blocks[:0]
        if not len(owners):
            continue
        cnt = np.ascontiguousarray(blocks[:, :4]).view(np.int32)[:, 0]
        ids = np.ascontiguousarray(blocks[:, 4: 4 + 4 * cap]).view(np.int32)
        live = (np.arange(cap)[None, :] < np.minimum(cnt, cap)[:, None]) & (ids >= 0)
        for v in owners[cnt > cap][:5]:
            bad.append(f"vertex {v} layer {layer}: degree above cap {cap}")
        for v in owners[((ids == owners[:, None]) & live).any(1)][:5]:
            bad.append(f"vertex {v} layer {layer}: self loop")
        out = live & (ids >= n)
        for v in owners[out.any(1)][:5]:
            bad.append(f"vertex {v} layer {layer}: neighbor id out of range")
        if layer:
            lv = np.where(live & ~out, graph.levels[np.clip(ids, 0, n - 1)], layer)
            for v in owners[(lv < layer).any(1)][:5]:
                bad.append(f"vertex {v} layer {layer}: neighbor below its layer")
    return bad
