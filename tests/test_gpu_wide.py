"""Wide vertex ids (n >= 2^24): 64-bit search keys with 32-bit tie ids,
32-bit visited-set slots and 64-bit global-tier entries (FlashDistW /
ExactDistW, search.cuh).

* forced on a small graph (FLASHANN_B200_WIDE=1) the wide kernels build the
  same graph as the oracle row for row — tie order 0 (vertex id) and the
  salted scramble over 32-bit tie ids (oracle tie mode 4), with the global
  visited tier forced (hash_log2 = 9) — and search it bit-exactly;
* the exact kind (kind 0) too;
* at n = 2^24 + 10^5 (past the narrow kernels' range) the build selects the
  wide kernels by itself and produces a valid graph whose rows reach ids
  >= 2^24, and queries find their own base vectors.
"""

import os

import numpy as np
import pytest

import golden_inputs as gi
from oracle import native

pytestmark = pytest.mark.gpu


@pytest.fixture
def wide_env():
    os.environ["FLASHANN_B200_WIDE"] = "1"
    yield
    os.environ.pop("FLASHANN_B200_WIDE", None)


def _prov(golden, codes=None):
    dmin, delta = golden["g_range"]
    data, _ = gi.graph_data()
    return {"vecs": data, "dim": data.shape[1], "proj": golden["g_proj"],
            "codes": (golden["g_codes"] if codes is None else codes).copy(),
            "cent": golden["g_cent"], "dims": golden["g_dims"], "offs": golden["g_offs"],
            "sdt": golden["g_sdt"], "dist_min": float(dmin), "delta": float(delta)}


SCHED = {"sequential": dict(batch_max=1, batch_frac=1.0, seq_prefix=1 << 30),
         "default": dict(batch_max=4096, batch_frac=0.1, seq_prefix=0)}


@pytest.mark.parametrize("hash_log2", [0, 9])
@pytest.mark.parametrize("tie", [0, 2])
@pytest.mark.parametrize("sched", list(SCHED))
def test_wide_build_matches_oracle(cuda, golden, wide_env, sched, tie, hash_log2):
    from paper_2502_18113_b200 import layout, sm100

    g = gi.GRAPH
    prov = _prov(golden, codes=np.zeros_like(golden["g_codes"]))
    levels, uoff = golden["g_levels"], golden["g_uoff"]
    R, m = g["R"], prov["cent"].shape[0]
    base = layout.empty_rows(len(levels), 2 * R, m)
    upper = layout.empty_rows(int(levels.sum()), R, m)
    opts = SCHED[sched]
    saved = dict(sm100.BUILD_OPTIONS)
    sm100.BUILD_OPTIONS.update(opts, hash_log2=hash_log2, tie=tie, expand=1)
    try:
        res = sm100.build_graph(4, prov, levels, base, uoff, upper, g["C"], R)
    finally:
        sm100.BUILD_OPTIONS.clear()
        sm100.BUILD_OPTIONS.update(saved)
    # oracle tie 4 = the salted scramble over 32-bit tie ids
    hg = native.HostGraph(levels, uoff, R, m, tie={0: 0, 2: 4}[tie], expand=1)
    ores = hg.build(prov["proj"], prov["cent"], prov["dims"], prov["offs"], prov["dist_min"],
                    prov["delta"], prov["sdt"], g["C"], **opts)
    assert (res["entry_point"], res["max_layer"]) == (ores["entry_point"], ores["max_layer"])
    for v in range(len(levels)):
        assert np.array_equal(layout.row_ids(base, v, 2 * R), hg.neighbors(v, 0)), v
        for lay in range(1, levels[v] + 1):
            r = uoff[v] + lay - 1
            assert np.array_equal(layout.row_ids(upper, r, R), hg.neighbors(v, lay)), (v, lay)
    for k in ("dist_comps", "visited", "kernel_calls"):
        assert res["counters"][k] == ores["counters"][k], k
    # query search on the built graph (tie order 0), with and without rerank
    hq = native.HostGraph.from_blocks(levels, uoff, base, upper, R, prov["codes"])
    queries = gi.graph_data()[1]
    qaux = golden["g_qproj"]
    e, ml = res["entry_point"], res["max_layer"]
    for rr in (0, 16):
        ids, ds, _ = sm100.search_batch(4, prov, levels, base, uoff, upper, g["C"], R, e, ml,
                                        queries, qaux, g["ef"], 10, rr)
        oid, od, _ = hq.search(prov["vecs"], prov["cent"], prov["dims"], prov["offs"],
                               prov["dist_min"], prov["delta"], e, ml, queries, qaux, g["ef"],
                               10, rr)
        assert np.array_equal(ids, oid) and np.array_equal(ds, od), rr


def test_wide_exact_kind_matches_oracle(cuda, wide_env):
    from paper_2502_18113_b200 import graph, layout, sm100

    rng = np.random.default_rng(11)
    n, dim, R, C_ = 1500, 12, 6, 40
    vecs = rng.normal(size=(n, dim)).astype(np.float32)
    levels = graph.assign_layers(n, 3, R)
    uoff = graph.upper_offsets_of(levels)
    base = layout.empty_rows(n, 2 * R, 0)
    upper = layout.empty_rows(int(levels.sum()), R, 0)
    saved = dict(sm100.BUILD_OPTIONS)
    sm100.BUILD_OPTIONS.update(SCHED["default"], tie=0, expand=1)
    try:
        res = sm100.build_graph(0, {"vecs": vecs, "dim": dim}, levels, base, uoff, upper, C_, R)
    finally:
        sm100.BUILD_OPTIONS.clear()
        sm100.BUILD_OPTIONS.update(saved)
    hg = native.HostGraph(levels, uoff, R, 0, tie=0, expand=1, kind=0, vecs=vecs)
    ores = hg.build_exact(C_, **SCHED["default"])
    assert (res["entry_point"], res["max_layer"]) == (ores["entry_point"], ores["max_layer"])
    for v in range(n):
        assert np.array_equal(layout.row_ids(base, v, 2 * R), hg.neighbors(v, 0)), v


def test_wide_ids_past_2_24(cuda):
    """n = 2^24 + 100,000: the index picks the wide kernels on its own."""
    torch = cuda
    from paper_2502_18113_b200 import builder, flash, graph

    n, dim = (1 << 24) + 100_000, 16
    gen = torch.Generator(device="cuda").manual_seed(5)
    centres = torch.randn((256, dim), generator=gen, device="cuda")
    x = centres[torch.randint(0, 256, (n,), generator=gen, device="cuda")]
    x += 0.3 * torch.randn((n, dim), generator=gen, device="cuda")
    sample = x[:: n // 20000][:20000].contiguous()
    model = flash.flash_train(sample, dim, 8, seed=0, kmeans_iters=5)
    params = graph.BuildParams(C=24, R=6, seed=0)
    levels = graph.assign_layers(n, 0, params.R)
    prov = flash.FlashProvider(model)
    prov.attach(x, vecs_dev=x)
    g = graph.GraphIndex(n, dim, params, "flash", model.m, levels)
    ctr = builder.build_device(g, prov, params)
    assert ctr["n_batches"] > 0
    from paper_2502_18113_b200 import _lib

    lib = _lib.load()
    cap = 2 * params.R
    rows0 = torch.empty((n, 1 + cap), dtype=torch.int32, device="cuda")
    rowsU = torch.empty((max(g.n_upper_rows, 1), 1 + params.R), dtype=torch.int32, device="cuda")
    _lib.check(lib.fa_index_export_rows(g.handle, rows0.data_ptr(), rowsU.data_ptr(), None))
    torch.cuda.synchronize()
    cnt0, ids0 = rows0[:, 0], rows0[:, 1:]
    live = ids0 >= 0
    assert torch.equal(live.sum(1).to(torch.int32), cnt0)
    assert int(cnt0.min()) >= 1 and int(cnt0.max()) <= cap
    assert int(ids0.max()) < n and int(ids0.max()) >= (1 << 24)
    self_loop = (ids0 == torch.arange(n, device="cuda", dtype=torch.int32)[:, None]).any()
    assert not bool(self_loop)
    # the vertices past 2^24 are wired in like their predecessors: the share
    # with incoming edges matches the 100K ids just below 2^24 (pruning under
    # coarse 4-bit codes leaves some late vertices without in-edges either way)
    indeg = torch.bincount(ids0[live].long(), minlength=n)
    lo = float((indeg[(1 << 24) - 100_000: 1 << 24] > 0).float().mean())
    hi = float((indeg[1 << 24:] > 0).float().mean())
    assert hi >= 0.5 and abs(hi - lo) <= 0.1, (lo, hi)
    # vertices past 2^24 are found by search as often as those just below:
    # queries equal to base vectors, Flash search + exact rerank
    from paper_2502_18113_b200 import evaluation

    def self_hits(first):
        qi = torch.arange(first, first + 2000, 4, device="cuda")
        ids, _, _ = evaluation.search_batch_dev(
            g, prov, x[qi].contiguous(), evaluation.SearchParams(ef=128, k=10, rerank_depth=128))
        return float((ids.cpu().numpy() == qi.cpu().numpy()[:, None]).any(1).mean())

    below, above = self_hits((1 << 24) - 2000), self_hits(n - 2000)
    assert above > 0.1 and abs(above - below) <= 0.15, (below, above)
