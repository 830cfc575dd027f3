"""Drop-in cases run INSIDE the reference's test tree (TEST INFRASTRUCTURE).

tests/test_gpu_reference_suite.py copies this file next to the reference's own
tests as test_sm100_dropin.py and runs it with the sm100 core injected
(sm100_inject.py).  Everything goes through the reference's public API —
``flashann.build(..., core_impl=...)`` (builder.py:88-120) and
``flashann.evaluation.search_batch(..., core_impl=...)`` (evaluation.py:72-89)
— and is compared with the reference's semantic core (_pycore), whose
(d, id) rules the GPU core restates exactly at batch size 1 and tie order 0.
"""

from contextlib import contextmanager

import numpy as np
import pytest

from flashann import _pycore, core
from flashann.builder import StrategyParams, build
from flashann.dataset import VectorDataset, brute_force_knn, gen_synthetic
from flashann.evaluation import SearchParams, recall_at_k, search_batch
from flashann.graph import BuildParams, check_invariants
from paper_2502_18113_b200 import sm100

SEQUENTIAL = dict(batch_max=1, batch_frac=1.0, seq_prefix=1 << 30, tie=0, expand=1)


@contextmanager
def build_options(**kw):
    saved = dict(sm100.BUILD_OPTIONS)
    sm100.BUILD_OPTIONS.update(kw)
    try:
        yield
    finally:
        sm100.BUILD_OPTIONS.clear()
        sm100.BUILD_OPTIONS.update(saved)


def _same_graph(a, b):
    assert (a.entry_point, a.max_layer) == (b.entry_point, b.max_layer)
    for layer in range(a.max_layer + 1):
        for v in np.flatnonzero(a.levels >= layer):
            assert np.array_equal(a.neighbors(int(v), layer), b.neighbors(int(v), layer)), \
                (layer, int(v))


def test_core_is_injected():
    assert core.HAVE_EXT and core.active_core() is sm100 and core.core_name() == "sm100"
    # every reference kernel name resolves without a registry patch
    for name in ("auto", "scalar", "vector128", "vector256", "vector512"):
        assert 0 <= core.resolve_kernel(name) <= 3


@pytest.fixture(scope="module")
def flash_pair():
    ds = gen_synthetic(400, 24, 6, seed=5)
    params = BuildParams(C=24, R=4, seed=5)
    sp = StrategyParams(m_f=8, d_f=24, kmeans_iters=10)
    ref = build(ds, "flash", params, sp, core_impl=_pycore)
    with build_options(**SEQUENTIAL):
        gpu = build(ds, "flash", params, sp, core_impl=sm100)
    return ds, ref, gpu


def test_flash_sequential_build_equals_semantic_core(flash_pair):
    """reference build() through sm100 (batch 1, tie 0) == build() through _pycore."""
    _, ref, gpu = flash_pair
    assert np.array_equal(ref.provider.core_arrays()["codes"], gpu.provider.core_arrays()["codes"])
    _same_graph(ref.graph, gpu.graph)


def test_flash_search_equals_semantic_core(flash_pair):
    """reference search_batch() through sm100 == through _pycore, same graph."""
    ds, ref, _ = flash_pair
    rng = np.random.default_rng(6)
    queries = ds.data[rng.choice(ds.n, 40, replace=False)] + 0.01
    for ef in (10, 32, 100):
        a = search_batch(ref.graph, ref.provider, queries, SearchParams(ef=ef, k=10),
                         core_impl=_pycore)
        b = search_batch(ref.graph, ref.provider, queries, SearchParams(ef=ef, k=10),
                         core_impl=sm100)
        assert np.array_equal(a[0], b[0]), ef
        assert np.array_equal(a[1], b[1]), ef


def test_flash_default_build_through_reference_api():
    """The default (batched) GPU schedule through build(): a valid index whose
    recall matches the semantic core's sequential graph on the same data."""
    ds = gen_synthetic(3000, 32, 16, seed=11)
    params = BuildParams(C=64, R=8, seed=11)
    sp = StrategyParams(m_f=8, d_f=32)
    gpu = build(ds, "flash", params, sp, core_impl=sm100)
    assert check_invariants(gpu.graph, gpu.provider, heuristic_sample=50) == []
    queries = ds.data[:200]
    gt = brute_force_knn(ds, VectorDataset(queries), 10)
    ids, _, _ = search_batch(gpu.graph, gpu.provider, queries,
                             SearchParams(ef=64, k=10, rerank_depth=64), core_impl=sm100)
    assert recall_at_k(ids, gt) >= 0.5


def test_exact_build_and_wide_search_through_reference_api():
    """kind 0 through build()/search_batch(): a wide (ef > 512) search finds
    the true nearest neighbour of base points."""
    ds = gen_synthetic(1500, 16, 8, seed=12)
    res = build(ds, "exact", BuildParams(C=40, R=6, seed=12), core_impl=sm100)
    assert check_invariants(res.graph, res.provider, heuristic_sample=30) == []
    queries = ds.data[:50]
    ids, dists, _ = search_batch(res.graph, res.provider, queries, SearchParams(ef=1500, k=1),
                                 core_impl=sm100)
    assert (ids[:, 0] == np.arange(50)).all()
    assert (dists[:, 0] == 0.0).all()
