"""End-to-end index construction (mirrors flashann/builder.py:34-120).

`build(dataset, "flash", BuildParams, StrategyParams)` trains the coder on a
bounded sample, projects + encodes every vector, draws the layers and runs
the batched-insertion build — all on the GPU, with the same timing split as
the reference: coding_seconds = sample + train, graph_seconds = attach +
levels + alloc + build.  Passing `core_impl=` runs the reference-shaped
host-array contract instead (e.g. the sm100 core or the reference's own
compiled core), exactly like the reference's builder.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib, graph, layout
from ._arrays import rows_of
from ._lib import check
from .errors import ConfigError
from .flash import FlashProvider, flash_train

STRATEGIES = ("flash",)
DEFAULT_SAMPLE = 100_000


@dataclass
class StrategyParams:
    m_pq: int = 16
    l_pq: int = 8
    l_sq: int = 8
    alpha: float = 0.9
    m_f: int = 16
    d_f: int | None = None
    kmeans_iters: int = 25


@dataclass
class BuildResult:
    graph: graph.GraphIndex
    provider: FlashProvider
    coding_seconds: float
    graph_seconds: float
    counters: dict = field(default_factory=dict)

    @property
    def total_seconds(self) -> float:
        return self.coding_seconds + self.graph_seconds


def training_sample(dataset, sample_size: int, seed: int):
    """<= sample_size rows drawn without replacement, sorted (builder.py:60-65)."""
    data = rows_of(dataset)
    n = data.shape[0]
    if n <= sample_size:
        return data
    rng = np.random.default_rng(seed)
    sel = np.sort(rng.choice(n, size=sample_size, replace=False))
    return data[sel]


def train_provider(strategy: str, sample, sp: StrategyParams, seed: int = 0):
    if strategy == "exact":
        from .exact import ExactProvider

        return ExactProvider()
    if strategy != "flash":
        raise ConfigError(f"strategy {strategy!r} is outside this GPU core ('flash', 'exact')")
    d_f = sp.d_f
    if d_f is None:
        from .pca import pca_train

        d_f = max(pca_train(sample, alpha=sp.alpha).d, sp.m_f)
    return FlashProvider(flash_train(sample, d_f, sp.m_f, seed=seed,
                                     kmeans_iters=sp.kmeans_iters))


def build_options(params: graph.BuildParams, start: int = 0, end: int = 0,
                  **overrides) -> _lib.BuildOpts:
    from . import sm100

    o = dict(sm100.BUILD_OPTIONS)
    o.update(overrides)
    return _lib.BuildOpts(C=params.C, batch_max=o["batch_max"], batch_frac=o["batch_frac"],
                          seq_prefix=o["seq_prefix"], hash_log2=o["hash_log2"],
                          profile=o.get("profile", 0), tie=o.get("tie", 2),
                          expand=o.get("expand", 1), batch_min=o.get("batch_min", -1),
                          start=int(start), end=int(end))


def build_device(g: graph.GraphIndex, provider: FlashProvider, params: graph.BuildParams,
                 stream=None, start: int = 0, end: int = 0, **overrides) -> dict:
    """Batched insertion on the device index of `g`: every vertex, or the
    range [start, end) — start > 0 resumes the graph the earlier calls built
    (vertices [0, start)), the dynamic-rebuild workload of BASELINE config 5."""
    from .sm100 import check_limits

    lib = _lib.load()
    check_limits(g.n, params.C, params.R, provider.code_subspaces)
    if g.handle is None:
        g.create_device(provider)
    res = _lib.BuildResult()
    opts = build_options(params, start=start, end=end, **overrides)
    check(lib.fa_index_build(g.handle, C.byref(opts), C.byref(res), stream))
    g.entry_point = int(res.entry_point)
    g.max_layer = int(res.max_layer)
    g.counters = dict(res.counters(), reverse_prunes=int(res.reverse_prunes),
                      reverse_appends=int(res.reverse_appends), n_batches=int(res.n_batches),
                      reverse_full_prunes=int(res.reverse_full_prunes),
                      launches=int(res.launches), ms_encode=res.ms_encode,
                      ms_search=res.ms_search, ms_sort=res.ms_sort, ms_reverse=res.ms_reverse)
    g.invalidate()
    return g.counters


def build(dataset, strategy: str, params: graph.BuildParams, sp: StrategyParams | None = None,
          sample_size: int = DEFAULT_SAMPLE, kernel: str | None = None,
          core_impl=None) -> BuildResult:
    """Train, encode, and insert the whole dataset."""
    data = rows_of(dataset)
    n = data.shape[0]
    if n < 1:
        raise ConfigError("cannot build an index over an empty dataset")
    sp = sp or StrategyParams()
    import torch

    t0 = time.perf_counter()
    sample = training_sample(dataset, sample_size, params.seed)
    provider = train_provider(strategy, sample, sp, seed=params.seed)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    provider.attach(dataset)
    levels = graph.assign_layers(n, params.seed, params.R)
    g = graph.GraphIndex(n, data.shape[1], params, strategy, provider.code_subspaces, levels)
    if core_impl is None:
        build_device(g, provider, params)
    else:
        # reference-shaped host contract (_core.pyx:711-764)
        pv = provider.core_arrays()
        base = layout.empty_rows(n, 2 * params.R, provider.code_subspaces)
        upper = layout.empty_rows(g.n_upper_rows, params.R, provider.code_subspaces)
        out = core_impl.build_graph(provider.kind_id, pv, g.levels, base, g.upper_offsets,
                                    upper, params.C, params.R, threads=params.threads, kernel=0)
        g.entry_point, g.max_layer = int(out["entry_point"]), int(out["max_layer"])
        g.counters = dict(out["counters"])
        g._blocks = (base, upper)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return BuildResult(graph=g, provider=provider, coding_seconds=t1 - t0,
                       graph_seconds=t2 - t1, counters=g.counters)
