"""GPU exact strategy (kind 0): fp32-L2 build and search
against the reference's semantic core (golden, tests/golden/gen_exact_golden.py)
and the oracle's batched exact build."""

from pathlib import Path

import numpy as np
import pytest

from oracle import native

pytestmark = pytest.mark.gpu

G = Path(__file__).resolve().parent / "golden" / "exact_golden.npz"


@pytest.fixture(scope="module")
def core(cuda):
    from paper_2502_18113_b200 import sm100

    return sm100


def _golden():
    g = dict(np.load(G))
    return g, tuple(int(x) for x in g["params"])


def _build(core, vecs, levels, uoff, R, C, **opts):
    from paper_2502_18113_b200 import layout

    base = layout.empty_rows(len(levels), 2 * R, 0)
    upper = layout.empty_rows(int(levels.sum()), R, 0)
    saved = dict(core.BUILD_OPTIONS)
    core.BUILD_OPTIONS.update(opts)
    try:
        res = core.build_graph(0, {"vecs": vecs, "dim": vecs.shape[1]}, levels, base, uoff,
                               upper, C, R)
    finally:
        core.BUILD_OPTIONS.clear()
        core.BUILD_OPTIONS.update(saved)
    return res, base, upper


def test_exact_sequential_build_matches_reference(core):
    from paper_2502_18113_b200 import layout

    g, (R, C, ef, k) = _golden()
    res, base, upper = _build(core, g["vecs"], g["levels"], g["uoff"], R, C, batch_max=1,
                              batch_frac=1.0, seq_prefix=1 << 30, tie=0)
    assert (res["entry_point"], res["max_layer"]) == tuple(int(x) for x in g["state"])
    for v in range(len(g["levels"])):
        assert np.array_equal(layout.row_ids(base, v, 2 * R), layout.row_ids(g["base"], v, 2 * R)), v
        for lay in range(1, g["levels"][v] + 1):
            r = g["uoff"][v] + lay - 1
            assert np.array_equal(layout.row_ids(upper, r, R), layout.row_ids(g["upper"], r, R))


def test_exact_search_matches_reference(core):
    g, (R, C, ef, k) = _golden()
    e, ml = (int(x) for x in g["state"])
    prov = {"vecs": g["vecs"], "dim": g["vecs"].shape[1]}
    ids, d, _ = core.search_batch(0, prov, g["levels"], g["base"], g["uoff"], g["upper"], C, R, e,
                                  ml, g["queries"], None, ef, k, 0)
    assert np.array_equal(ids, g["ids"]) and np.array_equal(d, g["d"])


@pytest.mark.parametrize("tie", [0, 2])
def test_exact_batched_build_matches_oracle(core, tie):
    from paper_2502_18113_b200 import graph, layout

    rng = np.random.default_rng(31 + tie)
    n, dim, R, C = 2500, 24, 8, 48
    x = (rng.normal(size=(12, dim))[rng.integers(0, 12, n)] + 0.4 * rng.normal(size=(n, dim)))
    x = x.astype(np.float32)
    levels = graph.assign_layers(n, 3, R)
    uoff = graph.upper_offsets_of(levels)
    sched = dict(batch_max=256, batch_frac=0.2, seq_prefix=16)
    res, base, upper = _build(core, x, levels, uoff, R, C, tie=tie, **sched)
    hg = native.HostGraph(levels, uoff, R, 0, kind=0, vecs=x, tie=tie)
    o = hg.build_exact(C, **sched)
    assert (res["entry_point"], res["max_layer"]) == (o["entry_point"], o["max_layer"])
    for v in range(n):
        assert np.array_equal(layout.row_ids(base, v, 2 * R), hg.neighbors(v, 0)), v
        for lay in range(1, levels[v] + 1):
            r = uoff[v] + lay - 1
            assert np.array_equal(layout.row_ids(upper, r, R), hg.neighbors(v, lay))
    for key in ("dist_comps", "visited"):
        assert res["counters"][key] == o["counters"][key], key
    q = rng.normal(size=(30, dim)).astype(np.float32)
    prov = {"vecs": x, "dim": dim}
    ids, d, _ = core.search_batch(0, prov, levels, base, uoff, upper, C, R, res["entry_point"],
                                  res["max_layer"], q, None, 32, 10, 0)
    hq = native.HostGraph.from_blocks(levels, uoff, base, upper, R, None, kind=0, vecs=x)
    oi, od, _ = hq.search_exact(res["entry_point"], res["max_layer"], q, 32, 10)
    assert np.array_equal(ids, oi) and np.array_equal(d, od)


def test_exact_high_level_build_and_search(core):
    """builder.build(..., "exact") on the device index == the host drop-in."""
    from paper_2502_18113_b200 import builder, evaluation, graph, layout

    rng = np.random.default_rng(8)
    x = (rng.normal(size=(10, 32))[rng.integers(0, 10, 3000)]
         + 0.3 * rng.normal(size=(3000, 32))).astype(np.float32)
    params = graph.BuildParams(C=40, R=8, seed=2)
    res = builder.build(x, "exact", params)
    g = res.graph
    out, base, upper = _build(core, x, g.levels, g.upper_offsets, 8, 40)
    assert (g.entry_point, g.max_layer) == (out["entry_point"], out["max_layer"])
    for v in range(3000):
        assert np.array_equal(g.neighbors(v, 0), layout.row_ids(base, v, 16)), v
    q = rng.normal(size=(25, 32)).astype(np.float32)
    ids, d, _ = evaluation.search_batch(g, res.provider, q, evaluation.SearchParams(ef=24, k=6))
    ids2, d2, _ = core.search_batch(0, {"vecs": x, "dim": 32}, g.levels, base, g.upper_offsets,
                                    upper, 40, 8, out["entry_point"], out["max_layer"], q, None,
                                    24, 6, 0)
    assert np.array_equal(ids, ids2) and np.array_equal(d, d2)
