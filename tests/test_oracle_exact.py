"""Oracle pin for the exact strategy (kind 0): the oracle's sequential exact
build and search equal the reference semantic core's (with the compiled fp32
distance; tests/golden/gen_exact_golden.py) row for row and bit for bit."""

from pathlib import Path

import numpy as np

from oracle import native
from paper_2502_18113_b200 import layout

G = Path(__file__).resolve().parent / "golden" / "exact_golden.npz"


def _golden():
    g = dict(np.load(G))
    return g, tuple(int(x) for x in g["params"])


def test_exact_sequential_build_matches_reference():
    g, (R, C, ef, k) = _golden()
    hg = native.HostGraph(g["levels"], g["uoff"], R, 0, kind=0, vecs=g["vecs"])
    res = hg.build_exact(C, batch_max=1, batch_frac=1.0, seq_prefix=1 << 30)
    assert (res["entry_point"], res["max_layer"]) == tuple(int(x) for x in g["state"])
    for v in range(len(g["levels"])):
        assert np.array_equal(layout.row_ids(g["base"], v, 2 * R), hg.neighbors(v, 0)), v
        for lay in range(1, g["levels"][v] + 1):
            r = g["uoff"][v] + lay - 1
            assert np.array_equal(layout.row_ids(g["upper"], r, R), hg.neighbors(v, lay))


def test_exact_search_matches_reference():
    g, (R, C, ef, k) = _golden()
    hq = native.HostGraph.from_blocks(g["levels"], g["uoff"], g["base"], g["upper"], R, None,
                                      kind=0, vecs=g["vecs"])
    e, ml = (int(x) for x in g["state"])
    ids, d, _ = hq.search_exact(e, ml, g["queries"], ef, k)
    assert np.array_equal(ids, g["ids"]) and np.array_equal(d, g["d"])
