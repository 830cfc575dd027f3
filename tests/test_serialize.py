"""FANNIDX1 index files against a file written by the
reference's own save_index (tests/golden/gen_index_golden.py)."""

from pathlib import Path

import numpy as np
import pytest

from oracle import native
from paper_2502_18113_b200 import layout, serialize
from paper_2502_18113_b200.errors import FormatError

GOLD = Path(__file__).resolve().parent / "golden" / "ref_index_small.fannidx"
GOLD_EXACT = Path(__file__).resolve().parent / "golden" / "ref_index_exact.fannidx"


@pytest.mark.parametrize("path,strategy", [(GOLD, "flash"), (GOLD_EXACT, "exact")])
def test_reader_and_writer_are_byte_exact(tmp_path, path, strategy):
    meta, sec = serialize.read_sections(path)
    assert meta["strategy"] == strategy and meta["n"] == 400 and meta["R"] == 8
    assert list(sec)[:5] == ["levels", "base_blocks", "upper_offsets", "upper_blocks", "vectors"]
    assert sec["base_blocks"].shape == (400, layout.block_stride(16, meta["code_subspaces"]))
    out = tmp_path / "copy.fannidx"
    serialize.write_sections(out, meta, sec)
    assert out.read_bytes() == path.read_bytes()


def test_rejects_bad_files(tmp_path):
    raw = GOLD.read_bytes()
    bad = tmp_path / "bad"
    bad.write_bytes(b"NOTANIDX" + raw[8:])
    with pytest.raises(FormatError, match="not an index file"):
        serialize.read_sections(bad)
    bad.write_bytes(raw[:8] + (2).to_bytes(4, "little") + raw[12:])
    with pytest.raises(FormatError, match="unsupported index version"):
        serialize.read_sections(bad)
    bad.write_bytes(raw[: len(raw) - 100])
    with pytest.raises(FormatError, match="truncated"):
        serialize.read_sections(bad)


def _live_rows(blocks, cap, m):
    return [(layout.row_ids(blocks, r, cap), layout.row_codes(blocks, r, cap, m))
            for r in range(blocks.shape[0])]


@pytest.mark.gpu
def test_device_round_trip(cuda, tmp_path):
    """Reference file -> device index -> file: every section equal, graph
    rows equal in their live slots (the reference leaves stale bytes in dead
    slots, _core.pyx:441-477), and the loaded index searches like the oracle
    over the same rows."""
    meta, sec = serialize.read_sections(GOLD)
    g, prov, ds = serialize.load_index(GOLD)
    assert (g.entry_point, g.max_layer) == (meta["entry_point"], meta["max_layer"])
    out = tmp_path / "rt.fannidx"
    g.invalidate()  # export from the device, not the cached host copy
    serialize.save_index(out, g, prov, ds)
    meta2, sec2 = serialize.read_sections(out)
    assert meta2 == meta
    m, R = meta["code_subspaces"], meta["R"]
    for name in sec:
        if name in ("base_blocks", "upper_blocks"):
            cap = 2 * R if name == "base_blocks" else R
            a, b = _live_rows(sec[name], cap, m), _live_rows(sec2[name], cap, m)
            assert all(np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1])
                       for x, y in zip(a, b)), name
        else:
            assert sec2[name].dtype == sec[name].dtype and np.array_equal(sec2[name], sec[name]), name
    # search over the loaded index == the oracle over the file's rows
    from paper_2502_18113_b200 import evaluation

    q = np.random.default_rng(4).normal(size=(20, 16)).astype(np.float32)
    ids, ds_, _ = evaluation.search_batch(g, prov, q, evaluation.SearchParams(ef=16, k=5))
    p = prov.core_arrays()
    hq = native.HostGraph.from_blocks(sec["levels"], sec["upper_offsets"], sec["base_blocks"],
                                      sec["upper_blocks"], R, sec["codes"])
    oid, od, _ = hq.search(p["vecs"], p["cent"], p["dims"], p["offs"], p["dist_min"],
                           p["delta"], g.entry_point, g.max_layer, q, prov.query_aux(q), 16, 5, 0)
    assert np.array_equal(ids, oid) and np.array_equal(ds_, od)


@pytest.mark.gpu
def test_exact_device_round_trip(cuda, tmp_path):
    """An exact-strategy file written by the reference: load on the device,
    write back identical sections, search like the oracle's exact searcher."""
    meta, sec = serialize.read_sections(GOLD_EXACT)
    g, prov, ds = serialize.load_index(GOLD_EXACT)
    out = tmp_path / "rt.fannidx"
    g.invalidate()
    serialize.save_index(out, g, prov, ds)
    meta2, sec2 = serialize.read_sections(out)
    assert meta2 == meta and list(sec2) == list(sec)
    for name in sec:
        if name in ("base_blocks", "upper_blocks"):
            cap = 2 * meta["R"] if name == "base_blocks" else meta["R"]
            for r in range(sec[name].shape[0]):
                assert np.array_equal(layout.row_ids(sec[name], r, cap),
                                      layout.row_ids(sec2[name], r, cap)), (name, r)
        else:
            assert np.array_equal(sec2[name], sec[name]), name
    from paper_2502_18113_b200 import evaluation

    q = np.random.default_rng(5).normal(size=(20, 16)).astype(np.float32)
    ids, d, _ = evaluation.search_batch(g, prov, q, evaluation.SearchParams(ef=16, k=5))
    hq = native.HostGraph.from_blocks(sec["levels"], sec["upper_offsets"], sec["base_blocks"],
                                      sec["upper_blocks"], meta["R"], None, kind=0,
                                      vecs=sec["vectors"])
    oi, od, _ = hq.search_exact(g.entry_point, g.max_layer, q, 16, 5)
    assert np.array_equal(ids, oi) and np.array_equal(d, od)
