"""CPU: the oracle's search/build semantics against the reference's semantic
core (flashann/_pycore.py), which defines the algorithm with ties broken by
vertex id (tuple order).  The encoder is pinned separately (test_oracle.py),
so here _pycore is fed the compiled core's fp32 encoder output to isolate the
graph algorithm.
"""

import numpy as np
import pytest

from oracle import native, refpkg

fa = refpkg.import_reference()
pytestmark = pytest.mark.skipif(fa is None, reason="reference not importable here")


def _random_flash_graph(rng, n, m, cap, ties=True):
    codes = rng.integers(0, 16, size=(n, m)).astype(np.uint8)
    if ties:  # few distinct code rows -> massive distance ties
        base = rng.integers(0, 16, size=(6, m))
        pick = rng.integers(0, 6, n)
        codes = base[pick].astype(np.uint8)
        flip = rng.random(codes.shape) < 0.1
        codes[flip] = rng.integers(0, 16, int(flip.sum()))
    adj = np.full((n, cap), -1, np.int32)
    cnt = np.zeros(n, np.int32)
    for v in range(n):
        k = int(rng.integers(1, cap + 1))
        nb = rng.choice(np.delete(np.arange(n), v), size=k, replace=False)
        adj[v, :k] = nb
        cnt[v] = k
    return codes, adj, cnt


@pytest.mark.parametrize("seed", range(6))
def test_layer_search_matches_pycore(seed):
    from paper_2502_18113_b200 import layout

    rng = np.random.default_rng(seed)
    n, m, R = 300, 8, 6
    cap = 2 * R
    codes, adj, cnt = _random_flash_graph(rng, n, m, cap, ties=seed % 2 == 0)
    base = layout.empty_rows(n, cap, m)
    for v in range(n):
        layout.set_row(base, v, cap, m, adj[v, : cnt[v]], codes[adj[v, : cnt[v]]])
    levels = np.zeros(n, np.int32)
    uoff = np.full(n, -1, np.int64)
    sdt = np.zeros((m, 16, 16), np.uint8)
    prov = {"vecs": np.zeros((n, 1), np.float32), "codes": codes, "sdt": sdt}
    hg = native.HostGraph.from_blocks(levels, uoff, base, layout.empty_rows(0, R, m), R, codes)
    w = fa._pycore.GraphWriter(4, prov, levels, base, uoff, layout.empty_rows(0, R, m), 64, R)
    for q in range(12):
        adt = rng.integers(0, 40 if seed % 2 == 0 else 256, size=(m, 16)).astype(np.uint8)
        entry = int(rng.integers(n))
        for width in (1, 4, 16, 64):
            ctx = {"vec": None, "code": None, "adt": adt}
            ref = w.greedy_search_layer(ctx, entry, width, 0)
            ids, ds, _ = hg.layer_search(adt, 0, entry, width)
            assert [u for u, _ in ref] == list(ids), (q, width)
            assert [d for _, d in ref] == list(ds.astype(float)), (q, width)


def test_sequential_build_matches_pycore(monkeypatch):
    """Batch size 1 everywhere = the reference's sequential build, bit-exact
    against _pycore.build_graph (same encoder outputs)."""
    from paper_2502_18113_b200 import graph, layout

    rng = np.random.default_rng(7)
    n, dim, R, C, m = 500, 16, 4, 24, 8
    data = rng.normal(size=(n, dim)).astype(np.float32)
    data[: n // 2] *= 0.1  # a dense blob -> ties
    model = fa.flash_train(fa.VectorDataset(data), d_f=16, m_f=m, seed=0, kmeans_iters=5)
    prov_obj = fa.FlashProvider(model)
    prov_obj.attach(fa.VectorDataset(data))
    pv = prov_obj.core_arrays()
    core = refpkg.load_ref_core()

    def fp32_encoder(cent, dims, offs, dmin, delta, reduced):
        return core.flash_encode_adt(cent, dims, offs, dmin, delta,
                                     np.asarray(reduced, np.float32))

    monkeypatch.setattr(fa._pycore, "flash_encode_adt", fp32_encoder)
    levels = graph.assign_layers(n, 3, R)
    uoff = graph.upper_offsets_of(levels)
    base = layout.empty_rows(n, 2 * R, m)
    upper = layout.empty_rows(int(levels.sum()), R, m)
    p1 = dict(pv, codes=pv["codes"].copy())
    out = fa._pycore.build_graph(4, p1, levels, base, uoff, upper, C, R)
    hg = native.HostGraph(levels, uoff, R, m)
    o2 = hg.build(pv["proj"], pv["cent"], pv["dims"], pv["offs"], pv["dist_min"], pv["delta"],
                  pv["sdt"], C, batch_max=1, batch_frac=1.0, seq_prefix=1 << 30)
    assert (out["entry_point"], out["max_layer"]) == (o2["entry_point"], o2["max_layer"])
    assert np.array_equal(p1["codes"], hg.codes)
    for v in range(n):
        assert list(layout.row_ids(base, v, 2 * R)) == list(hg.neighbors(v, 0)), v
        for lay in range(1, levels[v] + 1):
            r = uoff[v] + lay - 1
            assert list(layout.row_ids(upper, r, R)) == list(hg.neighbors(v, lay))
