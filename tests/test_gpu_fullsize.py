"""Properties of a full-size build (config 2: 1M x 128, M = 32, efC = 200) —
too large for the oracle, so size-independent checks: the reference's
structural invariants over every row and layer, every vertex linked, and the
graph's navigability measured the way the recall protocol does it (exact
search over the built adjacency, recall@10 against brute force; the
reference's own graph scores 0.22 here, profiles/r01_recall_parity_c2_1m.json)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_config2_full_build_properties(cuda):
    from paper_2502_18113_b200 import builder, dataset, graph, sm100
    from paper_2502_18113_b200.evaluation import recall_at_k

    c = dataset.CONFIGS[2]
    data, queries = dataset.baseline_config(2, nq=1000)
    res = builder.build(data, "flash", graph.BuildParams(C=c["efC"], R=c["M"], seed=0),
                        builder.StrategyParams(m_f=c["m_f"], d_f=c["d_f"], kmeans_iters=10))
    g = res.graph
    assert g.n == c["n"]
    assert graph.check_invariants(g) == []
    cnt0 = np.ascontiguousarray(g.base_blocks[:, :4]).view(np.int32)[:, 0]
    assert (cnt0 >= 1).all() and cnt0.max() <= 2 * c["M"]
    # navigability: exact-distance search over the Flash graph's adjacency
    gt = dataset.brute_force_knn(data, queries, 10)
    ids, d, _ = sm100.search_batch(0, {"vecs": data, "dim": data.shape[1]}, g.levels,
                                   g.base_blocks, g.upper_offsets, g.upper_blocks, c["efC"],
                                   c["M"], g.entry_point, g.max_layer, queries, None, 64, 10, 0)
    assert (np.diff(d, axis=1) >= 0).all()
    assert recall_at_k(ids, gt) > 0.2

