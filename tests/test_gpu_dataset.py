"""GPU ground truth (dataset.brute_force_knn) against the reference's
brute_force_knn (flashann/dataset.py:126-161).

* ids equal the reference's own output on the golden graph data (g_gt,
  written by tests/golden/gen_golden.py from the reference in the build
  container);
* distances equal a numpy restatement of the reference's float64 expanded
  form (_pairwise_sq, dataset.py:126-132) to 1e-9 relative;
* ties are ordered by ascending id (the reference's lexsort on (d, id)),
  including ties that straddle the k-th position and duplicated base rows.
"""

import numpy as np
import pytest

import golden_inputs as gi

pytestmark = pytest.mark.gpu


def _np_knn(base, queries, k):
    # restatement of dataset.py:126-161 with a full (d, id) sort
    q = queries.astype(np.float64)
    b = base.astype(np.float64)
    d2 = (q * q).sum(1)[:, None] + (b * b).sum(1)[None, :] - 2.0 * (q @ b.T)
    np.maximum(d2, 0.0, out=d2)
    ids = np.empty((q.shape[0], k), np.int64)
    ds = np.empty((q.shape[0], k))
    for i in range(q.shape[0]):
        o = np.lexsort((np.arange(b.shape[0]), d2[i]))[:k]
        ids[i], ds[i] = o, d2[i, o]
    return ids, ds


def test_knn_matches_reference_golden(cuda, golden):
    from paper_2502_18113_b200 import dataset

    data, queries = gi.graph_data()
    gt = dataset.brute_force_knn(data, queries, 10)
    assert np.array_equal(gt.ids, golden["g_gt"])
    _, ds = _np_knn(data, queries, 10)
    assert np.allclose(gt.dists, ds, rtol=1e-9, atol=1e-12)


def test_knn_ties_by_id(cuda):
    from paper_2502_18113_b200 import dataset

    rng = np.random.default_rng(3)
    # integer-valued coordinates: exact float64 distances, many exact ties
    base = rng.integers(0, 3, size=(3000, 4)).astype(np.float32)
    base[1500:1600] = base[:100]  # duplicated rows: ties by id across the set
    queries = rng.integers(0, 3, size=(64, 4)).astype(np.float32)
    for k in (1, 10, 300):
        gt = dataset.brute_force_knn(base, queries, k)
        ids, ds = _np_knn(base, queries, k)
        assert np.array_equal(gt.ids, ids), k
        assert np.array_equal(gt.dists, ds), k


def test_knn_block_independent_and_full_width(cuda):
    from paper_2502_18113_b200 import dataset

    rng = np.random.default_rng(4)
    base = rng.normal(size=(500, 12)).astype(np.float32)
    queries = rng.normal(size=(70, 12)).astype(np.float32)
    a = dataset.brute_force_knn(base, queries, 500, block=7)
    b = dataset.brute_force_knn(base, queries, 500, block=256)
    assert np.array_equal(a.ids, b.ids) and np.array_equal(a.dists, b.dists)
    ids, _ = _np_knn(base, queries, 500)
    assert np.array_equal(a.ids, ids)
