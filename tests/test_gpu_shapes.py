"""GPU build and search parity at the shapes of every BASELINE config.

The golden-graph tests pin one small shape.  Here each config's coder and
graph shape (m, R, C; config 4 through its 960 -> 256 PCA) is built on a
3,000-vector prefix of that config's synthetic data, by the GPU and by the
oracle under the same batch schedule, and compared row for row; the query
search over the result is compared too.  The shapes cover every kernel
variant the flagship configs select: register result sets of 4, 8 and 16
slots per lane (C = 100, 200/256, 300), the shared-memory result set
(C > 512), 2/3/4 ADT chunks (m = 32, 48, 64, 96) and 2/3 id-row chunks
(layer-0 cap 32, 64, 96).
"""

import numpy as np
import pytest

from oracle import native

pytestmark = pytest.mark.gpu

N = 3000
SCHED = dict(batch_max=512, batch_frac=0.2, seq_prefix=32)
# a schedule whose third batch is a full 65,536-vertex batch (1, 100, 10,100,
# 65,536, ...): the batch size of the production build
BIG = dict(batch_max=65536, batch_frac=100.0, seq_prefix=0)
SHAPES = {
    "c1": dict(cfg=1, C=None),
    "c2": dict(cfg=2, C=None),  # the bench's shape: m = 64 (4 ADT chunks), C = 200
    "c3": dict(cfg=3, C=None),
    "c4": dict(cfg=4, C=None),
    "c5": dict(cfg=5, C=None),
    "c1_wide": dict(cfg=1, C=600),  # W > 512: shared-memory result set
    "c2_batch64k": dict(cfg=2, C=None, n=80_000, sched=BIG),
}


@pytest.fixture(scope="module")
def core(cuda):
    from paper_2502_18113_b200 import sm100

    return sm100


def _setup(name):
    from paper_2502_18113_b200 import dataset, flash, graph

    spec = SHAPES[name]
    c = dataset.CONFIGS[spec["cfg"]]
    n = spec.get("n", N)
    data, queries = dataset.baseline_config(spec["cfg"], n=n, nq=50)
    model = flash.flash_train(data[:20_000], c["d_f"], c["m_f"], seed=0, kmeans_iters=4)
    prov = flash.FlashProvider(model)
    prov.attach(data)
    arrays = prov.core_arrays()
    qaux = prov.query_aux(queries)
    levels = graph.assign_layers(n, 0, c["M"])
    uoff = graph.upper_offsets_of(levels)
    C = spec["C"] or c["efC"]
    return c, data, queries, arrays, qaux, levels, uoff, C


@pytest.mark.parametrize("name", list(SHAPES))
def test_config_shape_build_and_search(core, name):
    from paper_2502_18113_b200 import layout

    c, data, queries, prov, qaux, levels, uoff, C = _setup(name)
    sched = SHAPES[name].get("sched", SCHED)
    n = levels.shape[0]
    R, m = c["M"], prov["cent"].shape[0]
    prov = dict(prov, codes=np.zeros_like(prov["codes"]))
    base = layout.empty_rows(n, 2 * R, m)
    upper = layout.empty_rows(int(levels.sum()), R, m)
    saved = dict(core.BUILD_OPTIONS)
    core.BUILD_OPTIONS.update(sched, tie=2, expand=1, hash_log2=0)
    try:
        res = core.build_graph(4, prov, levels, base, uoff, upper, C, R)
    finally:
        core.BUILD_OPTIONS.clear()
        core.BUILD_OPTIONS.update(saved)
    hg = native.HostGraph(levels, uoff, R, m, tie=2, expand=1)
    ores = hg.build(prov["proj"], prov["cent"], prov["dims"], prov["offs"], prov["dist_min"],
                    prov["delta"], prov["sdt"], C, **sched)
    assert (res["entry_point"], res["max_layer"]) == (ores["entry_point"], ores["max_layer"])
    assert np.array_equal(prov["codes"], hg.codes)
    if sched is BIG:
        assert ores["n_batches"] >= 4
    for v in range(n):
        assert np.array_equal(layout.row_ids(base, v, 2 * R), hg.neighbors(v, 0)), v
        for lay in range(1, levels[v] + 1):
            r = uoff[v] + lay - 1
            assert np.array_equal(layout.row_ids(upper, r, R), hg.neighbors(v, lay)), (v, lay)
    for k in ("dist_comps", "visited", "kernel_calls"):
        assert res["counters"][k] == ores["counters"][k], k

    # query search over the built graph (ties by id, as the reference searcher)
    hq = native.HostGraph.from_blocks(levels, uoff, base, upper, R, prov["codes"])
    e, ml = res["entry_point"], res["max_layer"]
    for rerank in (0, 32):
        ids, ds, _ = core.search_batch(4, prov, levels, base, uoff, upper, C, R, e, ml, queries,
                                       qaux, 64, 10, rerank)
        oid, od, _ = hq.search(prov["vecs"], prov["cent"], prov["dims"], prov["offs"],
                               prov["dist_min"], prov["delta"], e, ml, queries, qaux, 64, 10,
                               rerank)
        assert np.array_equal(ids, oid), rerank
        assert np.array_equal(ds, od), rerank
