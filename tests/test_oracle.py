"""CPU: the oracle restatement against the reference's golden outputs.

These pin the checker itself (oracle/oracle.c) before it is trusted by the
GPU parity tests.  Golden outputs come from the reference's compiled core and
trainer (tests/golden/gen_golden.py).
"""

import hashlib

import numpy as np
import pytest

import golden_inputs as gi
from oracle import native


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("d", gi.L2_DIMS)
def test_l2_tree_matches_reference(golden, d):
    a, b = gi.l2_inputs(d)
    got = np.array([native.l2sq_f32(x, y) for x, y in zip(a, b)])
    assert np.array_equal(got, golden[f"l2_{d}"])


def test_quantizer_matches_reference(golden):
    d, dmin, delta = gi.quantize_inputs()
    got = native.quantize(d, dmin, delta)
    assert np.array_equal(got, golden["quant"])
    # reference known answers (tests/test_flash.py:78-95)
    assert native.quantize(dmin, dmin, delta)[0] == 0
    assert native.quantize(dmin + delta, dmin, delta)[0] == 255
    assert native.quantize(dmin + delta / 2, dmin, delta)[0] == 127
    assert native.quantize(-1.0, dmin, delta)[0] == 0


@pytest.mark.parametrize("m", gi.SCAN_MS)
def test_scan_matches_reference(golden, m):
    adts, codes = gi.scan_cases(m)
    got = native.batch_many(adts, codes)
    assert np.array_equal(got[:256], golden[f"scan_{m}_head"])
    assert sha(got) == str(golden[f"scan_{m}_sha"])


def test_block_scan_matches_reference(golden):
    adt, flat = gi.block_case()
    assert np.array_equal(native.batch_lanes(adt, flat, 4), golden["blocks"])


@pytest.mark.parametrize("name", list(gi.MODELS))
def test_encoder_matches_reference(golden, name):
    p = f"model_{name}_"
    cent, dims, offs = golden[p + "cent"], golden[p + "dims"], golden[p + "offs"]
    dmin, dmax = golden[p + "range"]
    red = gi.encode_inputs(cent, dims, gi.MODELS[name])
    codes, adts = native.encode_adt(red, cent, dims, offs, dmin, dmax - dmin)
    assert np.array_equal(codes, golden[p + "enc_codes"])
    assert np.array_equal(adts, golden[p + "enc_adt"])
    red_u, dmins, deltas = gi.ulp_inputs(cent, dims, offs, gi.MODELS[name])
    for r in range(red_u.shape[0]):
        c, a = native.encode_adt(red_u[r], cent, dims, offs, dmins[r], deltas[r])
        assert np.array_equal(c[0], golden[p + "ulp_codes"][r])
        assert np.array_equal(a[0], golden[p + "ulp_adt"][r])


def test_sdt_and_select_match_reference(golden):
    sdt = golden["model_c1s_sdt"]
    codes = gi.select_codes(sdt.shape[0])
    a, b = gi.sdt_pairs(codes)
    got = np.array([native.sdt_sum(sdt, x, y) for x, y in zip(a, b)], np.int32)
    assert np.array_equal(got, golden["sdt_sums"])
    outs = []
    for ids, d, cap in gi.select_cases(codes, sdt):
        outs.append(np.array(native.select(sdt, codes, ids, d, cap) + [-2], np.int32))
    assert np.array_equal(np.concatenate(outs), golden["select_out"])


def test_trained_sdt_is_symmetric_with_zero_diagonal(golden):
    for name in gi.MODELS:
        sdt = golden[f"model_{name}_sdt"]
        assert np.array_equal(sdt, sdt.transpose(0, 2, 1))
        assert (np.einsum("ijj->ij", sdt) == 0).all()


def _golden_graph(golden):
    g = gi.GRAPH
    return native.HostGraph.from_blocks(golden["g_levels"], golden["g_uoff"], golden["g_base"],
                                        golden["g_upper"], g["R"], golden["g_codes"])


def test_oracle_search_on_reference_graph_is_order_free(golden):
    """(d, id) total order: the result does not depend on neighbour order."""
    hg = _golden_graph(golden)
    cent, dims, offs = golden["g_cent"], golden["g_dims"], golden["g_offs"]
    dmin, delta = golden["g_range"]
    _, adts = native.encode_adt(golden["g_qproj"][:20], cent, dims, offs, dmin, delta)
    rng = np.random.default_rng(0)
    base = [hg.layer_search(adts[q], 0, 0, 16) for q in range(20)]
    for r in range(hg.n):  # shuffle every live row in place
        c = hg.cnt0[r]
        hg.adj0[r, :c] = rng.permutation(hg.adj0[r, :c])
    for q in range(20):
        ids, ds, _ = hg.layer_search(adts[q], 0, 0, 16)
        assert np.array_equal(ids, base[q][0]) and np.array_equal(ds, base[q][1])


def test_oracle_search_matches_semantic_core_golden(golden):
    hg = _golden_graph(golden)
    cent, dims, offs = golden["g_cent"], golden["g_dims"], golden["g_offs"]
    dmin, delta = golden["g_range"]
    _, adts = native.encode_adt(golden["g_qproj"], cent, dims, offs, dmin, delta)
    expect = golden["py_search_ids"]
    off = 0
    for width in gi.PY_WIDTHS:
        for q in range(adts.shape[0]):
            ids, _, _ = hg.layer_search(adts[q], 0, int(golden["py_entries"][q]), width)
            row = expect[off: off + width]
            off += width
            assert list(ids) == [int(x) for x in row if x >= 0], (width, q)


def test_oracle_sequential_build_matches_semantic_core_golden(golden):
    from paper_2502_18113_b200 import layout

    pb = gi.PY_BUILD
    dmin, delta = golden["pb_range"]
    hg = native.HostGraph(golden["pb_levels"], golden["pb_uoff"], pb["R"],
                          golden["pb_cent"].shape[0])
    res = hg.build(golden["pb_proj"], golden["pb_cent"], golden["pb_dims"], golden["pb_offs"],
                   dmin, delta, golden["pb_sdt"], pb["C"], batch_max=1, batch_frac=1.0,
                   seq_prefix=1 << 30)
    assert [res["entry_point"], res["max_layer"]] == list(golden["pb_state"])
    assert np.array_equal(hg.codes, golden["pb_codes"])
    for v in range(pb["n"]):
        assert list(hg.neighbors(v, 0)) == list(layout.row_ids(golden["pb_base"], v, 2 * pb["R"]))


def test_schedule_properties():
    levels = np.zeros(5000, np.int32)
    levels[[0, 10, 300, 2000]] = [1, 2, 3, 1]
    st, sz = native.schedule(levels, 64, 0.05, 100)
    assert st[0] == 1 and sz.sum() == len(levels) - 1
    assert np.array_equal(np.concatenate([[1], (st + sz)[:-1]]), st)
    assert sz.max() <= 64
    assert (sz[st < 100] == 1).all()
    # a vertex raising the top layer is inserted alone
    for v in (10, 300):
        k = np.searchsorted(st, v)
        assert st[k] == v and sz[k] == 1


def test_flash_narrated_fixture_oracle_and_reference():
    from oracle import refpkg
    from paper_2502_18113_b200 import layout

    prov, levels, base, uoff, R = gi.flash_narrated()
    hg = native.HostGraph.from_blocks(levels, uoff, base, layout.empty_rows(0, R, 1), R,
                                      prov["codes"])
    _, adts = native.encode_adt(np.zeros(2, np.float32), prov["cent"], prov["dims"],
                                prov["offs"], prov["dist_min"], prov["delta"])
    ids, ds, c = hg.layer_search(adts[0], 0, 0, 4)
    assert list(ids) == [17, 5, 3, 9] and c["dist_comps"] == 7
    assert native.select(prov["sdt"], prov["codes"], ids, ds.astype(float), 2) == [17, 5]
    ref = refpkg.load_ref_core()
    if ref is None:
        pytest.skip("reference core not built")
    out, rc = ref.greedy_search_layer(4, prov, levels, base, uoff, layout.empty_rows(0, R, 1), 8,
                                      R, 0, 4, 0, np.zeros(2, np.float32),
                                      np.zeros(2, np.float32))
    assert [i for i, _ in out] == [17, 5, 3, 9] and rc["dist_comps"] == 7
    assert ref.select_neighbors(4, prov, list(ids), list(ds.astype(float)), 2) == [17, 5]
