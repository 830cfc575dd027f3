"""CPU: the numpy training restatement against the reference's golden models,
and the host-side helpers (layer draws, split_dims, layout rows)."""

import numpy as np
import pytest

import golden_inputs as gi
from oracle import train_np


@pytest.mark.parametrize("name", list(gi.MODELS))
def test_train_restatement_matches_reference(golden, name):
    spec = gi.MODELS[name]
    data = gi.model_data(spec)
    m = train_np.train(data, spec["d_f"], spec["m_f"], spec["seed"], spec["iters"])
    p = f"model_{name}_"
    assert np.array_equal(m["cent"], golden[p + "cent"])
    assert np.array_equal(m["sdt"], golden[p + "sdt"])
    assert (m["dist_min"], m["dist_max"]) == tuple(golden[p + "range"])


def test_split_dims_matches_restatement():
    from paper_2502_18113_b200.flash import split_dims

    for d, m in [(12, 4), (13, 5), (128, 64), (96, 48), (256, 64), (768, 96), (7, 7)]:
        a, b = split_dims(d, m)
        c, e = train_np.split_dims(d, m)
        assert np.array_equal(a, c) and np.array_equal(b, e)


def test_layer_draws_match_reference():
    from oracle import refpkg
    from paper_2502_18113_b200 import graph

    fa = refpkg.import_reference()
    if fa is None:
        pytest.skip("reference not importable here")
    for n, seed, R in [(1000, 0, 16), (5000, 7, 32), (777, 123456789, 2)]:
        assert np.array_equal(graph.assign_layers(n, seed, R), fa.assign_layers(n, seed, R))


def test_layout_rows_roundtrip_reference():
    from oracle import refpkg
    from paper_2502_18113_b200 import layout

    fa = refpkg.import_reference()
    if fa is None:
        pytest.skip("reference not importable here")
    import flashann.layout as rl

    rng = np.random.default_rng(3)
    for cap, m in [(32, 5), (16, 1), (64, 64), (96, 96)]:
        a = layout.empty_rows(3, cap, m)
        b = rl.alloc_blocks(3, cap, m)
        assert np.array_equal(a, b)
        for r, cnt in enumerate([0, cap // 3 + 1, cap]):
            ids = rng.integers(0, 10_000, cnt)
            codes = rng.integers(0, 16, (cnt, m)).astype(np.uint8)
            layout.set_row(a, r, cap, m, ids, codes)
            rl.write_vertex_block(b, r, cap, m, ids, codes)
            assert np.array_equal(a[r], b[r])
            assert np.array_equal(layout.row_codes(a, r, cap, m), codes)
            assert np.array_equal(layout.row_ids(a, r, cap), ids)


def test_workloads_prefix_stable():
    """baseline_config draws the same first rows (and queries) for every n, so
    a CPU prefix sample is exactly the start of the GPU arm's workload."""
    from paper_2502_18113_b200 import dataset

    for cfg in (1, 2, 3, 4, 5):
        a, qa = dataset.baseline_config(cfg, n=700, nq=20)
        b, qb = dataset.baseline_config(cfg, n=1500, nq=35)
        assert np.array_equal(a, b[:700]), cfg
        assert np.array_equal(qa, qb[:20]), cfg
        assert a.dtype == np.float32 and a.shape[1] == dataset.CONFIGS[cfg]["dim"]
    x5, _ = dataset.baseline_config(5, n=50, nq=0)
    assert np.array_equal(dataset._round_bf16(x5), x5)  # config 5 rows are bf16 values
