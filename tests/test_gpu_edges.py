"""GPU edge cases of the build and search entry points (the reference's own
edge behaviour: _core.pyx:726-728 empty build, :821-822 empty search, -1/+inf
padding of short results, :860-888), each checked against the oracle where
there is a graph to compare."""

import numpy as np
import pytest

from oracle import native

pytestmark = pytest.mark.gpu

R, C = 8, 32


@pytest.fixture(scope="module")
def core(cuda):
    from paper_2502_18113_b200 import sm100

    return sm100


@pytest.fixture(scope="module")
def model(cuda):
    from paper_2502_18113_b200 import flash

    rng = np.random.default_rng(5)
    sample = rng.normal(size=(600, 16)).astype(np.float32)
    return flash.flash_train(sample, 16, 8, seed=0, kmeans_iters=3)


def _arrays(model, data):
    from paper_2502_18113_b200 import flash

    p = flash.FlashProvider(model)
    p.attach(data)
    return p, p.core_arrays()


def _build(core, prov, n, seed=0, **sched):
    from paper_2502_18113_b200 import graph, layout

    m = prov["cent"].shape[0]
    levels = graph.assign_layers(n, seed, R)
    uoff = graph.upper_offsets_of(levels)
    base = layout.empty_rows(n, 2 * R, m)
    upper = layout.empty_rows(int(levels.sum()), R, m)
    saved = dict(core.BUILD_OPTIONS)
    core.BUILD_OPTIONS.update(sched)
    try:
        res = core.build_graph(4, prov, levels, base, uoff, upper, C, R)
    finally:
        core.BUILD_OPTIONS.clear()
        core.BUILD_OPTIONS.update(saved)
    return res, levels, uoff, base, upper


def _check_oracle(prov, levels, uoff, base, upper, res, tie=2, **sched):
    from paper_2502_18113_b200 import layout

    m = prov["cent"].shape[0]
    hg = native.HostGraph(levels, uoff, R, m, tie=tie)
    ores = hg.build(prov["proj"], prov["cent"], prov["dims"], prov["offs"], prov["dist_min"],
                    prov["delta"], prov["sdt"], C, **sched)
    assert (res["entry_point"], res["max_layer"]) == (ores["entry_point"], ores["max_layer"])
    for v in range(len(levels)):
        assert np.array_equal(layout.row_ids(base, v, 2 * R), hg.neighbors(v, 0)), v
        for lay in range(1, levels[v] + 1):
            assert np.array_equal(layout.row_ids(upper, uoff[v] + lay - 1, R),
                                  hg.neighbors(v, lay))


def test_empty_build_and_search(core, model):
    _, prov = _arrays(model, np.zeros((0, 16), np.float32))
    res, levels, uoff, base, upper = _build(core, prov, 0)
    assert res["entry_point"] == -1 and res["max_layer"] == -1
    assert all(v == 0 for v in res["counters"].values())
    q = np.zeros((3, 16), np.float32)
    with pytest.raises(ValueError, match="empty graph"):
        core.search_batch(4, prov, levels, base, uoff, upper, C, R, -1, -1, q,
                          np.zeros((3, 16), np.float32), 16, 5, 0)


@pytest.mark.parametrize("n", [1, 2, 3, 17])
def test_tiny_graphs(core, model, n):
    """Graphs smaller than a row and than ef: row-exact build, search padded
    with -1 / +inf past the reachable vertices."""
    rng = np.random.default_rng(n)
    data = rng.normal(size=(n, 16)).astype(np.float32)
    p, prov = _arrays(model, data)
    sched = dict(batch_max=4, batch_frac=0.5, seq_prefix=0)
    res, levels, uoff, base, upper = _build(core, prov, n, **sched)
    _check_oracle(prov, levels, uoff, base, upper, res, **sched)
    q = rng.normal(size=(4, 16)).astype(np.float32)
    k = n + 3
    qaux = p.query_aux(q)
    e, ml = res["entry_point"], res["max_layer"]
    ids, ds, _ = core.search_batch(4, prov, levels, base, uoff, upper, C, R, e, ml, q, qaux, 16,
                                   k, 0)
    hq = native.HostGraph.from_blocks(levels, uoff, base, upper, R, prov["codes"])
    oid, od, _ = hq.search(prov["vecs"], prov["cent"], prov["dims"], prov["offs"],
                           prov["dist_min"], prov["delta"], e, ml, q, qaux, 16, k, 0)
    assert np.array_equal(ids, oid) and np.array_equal(ds, od)
    assert ids.shape == (4, k)
    assert (ids[:, n:] == -1).all() and np.isinf(ds[:, n:]).all()
    assert np.isinf(ds[ids < 0]).all() and np.isfinite(ds[ids >= 0]).all()


def test_identical_vectors(core, model):
    """All distances tie: the tie order alone decides, still row-exact."""
    data = np.tile(np.random.default_rng(9).normal(size=(1, 16)).astype(np.float32), (400, 1))
    _, prov = _arrays(model, data)
    for tie in (0, 2):
        sched = dict(batch_max=64, batch_frac=0.1, seq_prefix=8)
        res, levels, uoff, base, upper = _build(core, dict(prov, codes=prov["codes"].copy()),
                                                400, tie=tie, **sched)
        _check_oracle(prov, levels, uoff, base, upper, res, tie=tie, **sched)


def test_single_batch_whole_graph(core, model):
    """One batch holding every vertex after the seed: all searches see only
    vertex 0 and the graph is built from reverse edges alone."""
    data = np.random.default_rng(3).normal(size=(300, 16)).astype(np.float32)
    _, prov = _arrays(model, data)
    sched = dict(batch_max=1 << 20, batch_frac=1e6, seq_prefix=0)
    res, levels, uoff, base, upper = _build(core, prov, 300, **sched)
    _check_oracle(prov, levels, uoff, base, upper, res, **sched)


@pytest.mark.parametrize("early", [1, 37, 299])
def test_late_projected_rows(core, model, early, monkeypatch):
    """The host drop-in uploads the projected vectors in two parts and the
    build waits for the second before the first batch that reads it
    (FLASHANN_B200_EARLY_ROWS moves the split): blocks, codes and result are
    byte-identical to a build whose rows all arrived first, and row-exact
    against the oracle."""
    data = np.random.default_rng(11).normal(size=(600, 16)).astype(np.float32)
    _, prov = _arrays(model, data)
    sched = dict(batch_max=64, batch_frac=0.2, seq_prefix=0)
    ref = _build(core, dict(prov, codes=prov["codes"].copy()), 600, **sched)
    monkeypatch.setenv("FLASHANN_B200_EARLY_ROWS", str(early))
    p2 = dict(prov, codes=prov["codes"].copy())
    res, levels, uoff, base, upper = _build(core, p2, 600, **sched)
    assert res["entry_point"] == ref[0]["entry_point"] and res["max_layer"] == ref[0]["max_layer"]
    assert res["counters"] == ref[0]["counters"]
    assert np.array_equal(base, ref[3]) and np.array_equal(upper, ref[4])
    _check_oracle(p2, levels, uoff, base, upper, res, **sched)


def test_resumed_build_equals_one_pass(cuda):
    """fa_build_opts.start / end (the dynamic-rebuild workload): inserting
    [0, A) and then resuming [A, n) gives the same graph as one pass, when A
    is a batch boundary of the one-pass schedule."""
    from oracle import native
    from paper_2502_18113_b200 import builder, flash, graph
    import golden_inputs as gi

    data, _ = gi.graph_data()
    n = data.shape[0]
    model = flash.flash_train(data, 32, 16, seed=0, kmeans_iters=4)
    params = graph.BuildParams(C=48, R=8, seed=0)
    levels = graph.assign_layers(n, 0, params.R)
    sched = dict(batch_max=128, batch_frac=0.2, seq_prefix=16, batch_min=0)
    starts, _ = native.schedule(levels, **sched)
    A = int(starts[len(starts) // 2])

    def rows(g):
        import torch
        from paper_2502_18113_b200 import _lib

        lib = _lib.load()
        r0 = torch.empty((n, 1 + 2 * params.R), dtype=torch.int32, device="cuda")
        rU = torch.empty((max(g.n_upper_rows, 1), 1 + params.R), dtype=torch.int32,
                         device="cuda")
        _lib.check(lib.fa_index_export_rows(g.handle, r0.data_ptr(), rU.data_ptr(), None))
        return r0.cpu().numpy(), rU.cpu().numpy()

    out = []
    for split in (None, A):
        prov = flash.FlashProvider(model)
        prov.attach(data)
        g = graph.GraphIndex(n, data.shape[1], params, "flash", model.m, levels)
        if split is None:
            builder.build_device(g, prov, params, **sched)
        else:
            builder.build_device(g, prov, params, end=split, **sched)
            builder.build_device(g, prov, params, start=split, **sched)
        out.append((rows(g), g.entry_point, g.max_layer))
        g.close()
    (a0, aU), ea, ma = out[0]
    (b0, bU), eb, mb = out[1]
    assert (ea, ma) == (eb, mb)
    assert np.array_equal(a0, b0)
    assert np.array_equal(aU, bU)
