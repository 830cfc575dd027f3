"""GPU parity of search and batched construction against the oracle.

* layer search / query search on a FIXED graph (the reference-built golden
  graph) are bit-exact against the (d, id) restatement in oracle/oracle.c;
* the batched GPU build equals the oracle's batched build row-for-row under
  the same schedule (and the fully sequential schedule is the (d, id)
  restatement of the reference's threads=1 build).
"""

import numpy as np
import pytest

import golden_inputs as gi
from oracle import native

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def core(cuda):
    from paper_2502_18113_b200 import sm100

    return sm100


def _prov(golden, codes=None):
    dmin, delta = golden["g_range"]
    data, _ = gi.graph_data()
    return {"vecs": data, "dim": data.shape[1], "proj": golden["g_proj"],
            "codes": (golden["g_codes"] if codes is None else codes).copy(),
            "cent": golden["g_cent"], "dims": golden["g_dims"], "offs": golden["g_offs"],
            "sdt": golden["g_sdt"], "dist_min": float(dmin), "delta": float(delta)}


def _oracle_graph(golden):
    return native.HostGraph.from_blocks(golden["g_levels"], golden["g_uoff"], golden["g_base"],
                                        golden["g_upper"], gi.GRAPH["R"], golden["g_codes"])


@pytest.mark.parametrize("width", [1, 4, 16, 48])
def test_layer_search_fixed_graph(core, golden, width):
    prov = _prov(golden)
    R = gi.GRAPH["R"]
    ix = core.DeviceIndex(prov, golden["g_levels"], golden["g_base"], golden["g_uoff"],
                          golden["g_upper"], R)
    hg = _oracle_graph(golden)
    qp = golden["g_qproj"]
    rng = np.random.default_rng(width)
    entries = rng.integers(0, hg.n, size=qp.shape[0])
    ids, ds, ns, ctr = ix.search_layer(qp, entries, width, 0)
    _, adts = native.encode_adt(qp, prov["cent"], prov["dims"], prov["offs"], prov["dist_min"],
                                prov["delta"])
    tot = 0
    for q in range(qp.shape[0]):
        oi, od, oc = hg.layer_search(adts[q], 0, int(entries[q]), width)
        assert ns[q] == len(oi)
        assert np.array_equal(ids[q, : ns[q]], oi), q
        assert np.array_equal(ds[q, : ns[q]], od.astype(np.float64)), q
        tot += oc["dist_comps"]
    assert ctr[0] == tot
    # upper layer: entries drawn from layer-1 members
    top = np.flatnonzero(golden["g_levels"] >= 1)
    if len(top):
        ent1 = top[rng.integers(0, len(top), size=qp.shape[0])]
        ids1, ds1, ns1, _ = ix.search_layer(qp, ent1, width, 1)
        for q in range(0, qp.shape[0], 5):
            oi, od, _ = hg.layer_search(adts[q], 1, int(ent1[q]), width)
            assert np.array_equal(ids1[q, : ns1[q]], oi)
    ix.close()


@pytest.mark.parametrize("rerank", [0, 32])
def test_query_search_fixed_graph(core, golden, rerank):
    prov = _prov(golden)
    g = gi.GRAPH
    data, queries = gi.graph_data()
    entry, ml = (int(x) for x in golden["g_state"])
    ids, ds, ctr = core.search_batch(4, prov, golden["g_levels"], golden["g_base"],
                                     golden["g_uoff"], golden["g_upper"], g["C"], g["R"], entry, ml,
                                     queries, golden["g_qproj"], g["ef"], 10, rerank)
    hg = _oracle_graph(golden)
    oid, od, oc = hg.search(data, prov["cent"], prov["dims"], prov["offs"], prov["dist_min"],
                            prov["delta"], entry, ml, queries, golden["g_qproj"], g["ef"], 10,
                            rerank)
    assert np.array_equal(ids, oid)
    assert np.array_equal(ds, od)
    assert ctr["dist_comps"] == oc["dist_comps"]
    assert ctr["visited"] == oc["visited"]


SCHEDULES = {
    "sequential": dict(batch_max=1, batch_frac=1.0, seq_prefix=1 << 30),
    "small": dict(batch_max=64, batch_frac=0.05, seq_prefix=64),
    "wide": dict(batch_max=512, batch_frac=0.5, seq_prefix=16),
    "default": dict(batch_max=4096, batch_frac=0.1, seq_prefix=0),
}


@pytest.mark.parametrize("hash_log2", [0, 9])
@pytest.mark.parametrize("expand", [1, 4, 8])
@pytest.mark.parametrize("tie", [0, 2])
@pytest.mark.parametrize("sched", list(SCHEDULES))
def test_batched_build_matches_oracle(core, golden, sched, tie, expand, hash_log2):
    """hash_log2 = 9 (512 shared slots) forces the global visited tier."""
    from paper_2502_18113_b200 import layout

    g = gi.GRAPH
    prov = _prov(golden, codes=np.zeros_like(golden["g_codes"]))
    levels, uoff = golden["g_levels"], golden["g_uoff"]
    R, m = g["R"], prov["cent"].shape[0]
    base = layout.empty_rows(len(levels), 2 * R, m)
    upper = layout.empty_rows(int(levels.sum()), R, m)
    opts = SCHEDULES[sched]
    saved = dict(core.BUILD_OPTIONS)
    core.BUILD_OPTIONS.update(opts, hash_log2=hash_log2, tie=tie, expand=expand)
    try:
        res = core.build_graph(4, prov, levels, base, uoff, upper, g["C"], R)
    finally:
        core.BUILD_OPTIONS.clear()
        core.BUILD_OPTIONS.update(saved)
    hg = native.HostGraph(levels, uoff, R, m, tie=tie, expand=expand)
    ores = hg.build(prov["proj"], prov["cent"], prov["dims"], prov["offs"], prov["dist_min"],
                    prov["delta"], prov["sdt"], g["C"], **opts)
    assert res["entry_point"] == ores["entry_point"]
    assert res["max_layer"] == ores["max_layer"]
    assert np.array_equal(prov["codes"], hg.codes)
    for v in range(len(levels)):
        got = layout.row_ids(base, v, 2 * R)
        assert np.array_equal(got, hg.neighbors(v, 0)), v
        assert np.array_equal(layout.row_codes(base, v, 2 * R, m), hg.codes[got])
        for lay in range(1, levels[v] + 1):
            r = uoff[v] + lay - 1
            assert np.array_equal(layout.row_ids(upper, r, R), hg.neighbors(v, lay)), (v, lay)
    oc = ores["counters"]
    for k in ("dist_comps", "visited", "kernel_calls"):
        assert res["counters"][k] == oc[k], k


def test_layer_search_matches_semantic_core(core, golden):
    """Bit-exact against the reference's semantic core (_pycore
    greedy_search_layer) on the reference-built graph (golden)."""
    prov = _prov(golden)
    ix = core.DeviceIndex(prov, golden["g_levels"], golden["g_base"], golden["g_uoff"],
                          golden["g_upper"], gi.GRAPH["R"])
    qp = golden["g_qproj"]
    expect = golden["py_search_ids"]
    off = 0
    for width in gi.PY_WIDTHS:
        ids, _, ns, _ = ix.search_layer(qp, golden["py_entries"], width, 0)
        for q in range(qp.shape[0]):
            row = expect[off: off + width]
            off += width
            assert list(ids[q, : ns[q]]) == [int(x) for x in row if x >= 0], (width, q)
    ix.close()


def test_sequential_build_matches_semantic_core(core, golden):
    """Batch size 1 = the reference's sequential build: every row equals the
    graph _pycore.build_graph built (golden, same encoder outputs)."""
    from paper_2502_18113_b200 import layout

    pb = gi.PY_BUILD
    dmin, delta = golden["pb_range"]
    prov = {"vecs": np.zeros((pb["n"], 1), np.float32), "proj": golden["pb_proj"],
            "codes": np.zeros_like(golden["pb_codes"]), "cent": golden["pb_cent"],
            "dims": golden["pb_dims"], "offs": golden["pb_offs"], "sdt": golden["pb_sdt"],
            "dist_min": float(dmin), "delta": float(delta)}
    levels, uoff = golden["pb_levels"], golden["pb_uoff"]
    R, m = pb["R"], prov["cent"].shape[0]
    base = layout.empty_rows(pb["n"], 2 * R, m)
    upper = layout.empty_rows(int(levels.sum()), R, m)
    saved = dict(core.BUILD_OPTIONS)
    core.BUILD_OPTIONS.update(SCHEDULES["sequential"], tie=0, expand=1)
    try:
        res = core.build_graph(4, prov, levels, base, uoff, upper, pb["C"], R)
    finally:
        core.BUILD_OPTIONS.clear()
        core.BUILD_OPTIONS.update(saved)
    assert [res["entry_point"], res["max_layer"]] == list(golden["pb_state"])
    assert np.array_equal(prov["codes"], golden["pb_codes"])
    for v in range(pb["n"]):
        assert np.array_equal(layout.row_ids(base, v, 2 * R),
                              layout.row_ids(golden["pb_base"], v, 2 * R)), v
    for r in range(upper.shape[0]):
        assert np.array_equal(layout.row_ids(upper, r, R), layout.row_ids(golden["pb_upper"], r, R))


def test_flash_narrated_trace(core):
    """Narrated fixture (Flash form): final set [17, 5, 3, 9] after exactly
    seven distance computations; pruning to 2 keeps [17, 5]."""
    from paper_2502_18113_b200 import layout

    prov, levels, base, uoff, R = gi.flash_narrated()
    out, ctr = core.greedy_search_layer(4, prov, levels, base, uoff, layout.empty_rows(0, R, 1),
                                        8, R, 0, 4, 0, np.zeros(2), np.zeros(2, np.float32))
    assert [i for i, _ in out] == [17, 5, 3, 9]
    assert ctr["dist_comps"] == 7
    kept = core.select_neighbors(4, prov, [c[0] for c in out], [c[1] for c in out], 2)
    assert kept == [17, 5]
