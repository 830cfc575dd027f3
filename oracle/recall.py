"""Recall@10 parity protocol — TEST/BASELINE INFRASTRUCTURE.

Same data, same trained coder, two graphs:
  * "reference": the reference's own compiled build_graph (oracle/_ref) on the
    host cores (threads = 1 is deterministic; all cores for large n);
  * "gpu": the batched sm100 build under its default (or a given) schedule.
Both graphs are searched by the SAME searcher — the reference's compiled
search_batch (_core.pyx:817-888) — as Flash (ef, k=10), Flash + rerank 64,
and exact-distance search over the same adjacency (kind 0).  Used by
tests/test_gpu_recall.py (config 1, driver-visible) and
scripts/recall_parity.py (configs 2-5 at full size or 1M prefixes).
"""

from __future__ import annotations

import time

import numpy as np

from . import refpkg


def recall_at_k(ids, gt_ids, k=10):
    hits = 0
    for row, truth in zip(ids, gt_ids):
        hits += len(set(int(i) for i in row[:k] if i >= 0) & set(int(t) for t in truth[:k]))
    return hits / (len(gt_ids) * k)


def build_pair(cfg, n, nq, seed, threads=1, schedules=None, ref=True, search_threads=None,
               kmeans_iters=None, data=None, queries=None):
    """-> {graph name: {"build_s", "flash", "rerank64", "exact"}} for one seed."""
    from paper_2502_18113_b200 import builder, dataset, flash, graph, layout, sm100

    c = dataset.CONFIGS[cfg]
    if data is None:
        data, queries = dataset.baseline_config(cfg, n=n, nq=nq)
    gt = dataset.brute_force_knn(data, queries, 10)
    sample = builder.training_sample(data, builder.DEFAULT_SAMPLE, seed)
    iters = kmeans_iters or 10
    model = flash.flash_train(sample, c["d_f"], c["m_f"], seed=seed, kmeans_iters=iters)
    prov0 = flash.FlashProvider(model)
    prov0.attach(data)
    pv = prov0.core_arrays()
    qaux = prov0.query_aux(queries)
    R, C = c["M"], c["efC"]
    levels = graph.assign_layers(n, seed, R)
    uoff = graph.upper_offsets_of(levels)
    m = model.m
    core = refpkg.load_ref_core()
    if core is None:
        raise RuntimeError("oracle/_ref reference core not built (make -C oracle ref)")
    kid = len(core.available_kernels()) - 1
    graphs = {}
    if ref:
        p = dict(pv, codes=pv["codes"].copy())
        base = layout.empty_rows(n, 2 * R, m)
        upper = layout.empty_rows(int(levels.sum()), R, m)
        t0 = time.perf_counter()
        out = core.build_graph(4, p, levels, base, uoff, upper, C, R, threads=threads,
                               kernel=kid)
        graphs["reference"] = (p, base, upper, out, time.perf_counter() - t0)
    for name, opts in (schedules or {"gpu": {}}).items():
        p = dict(pv, codes=pv["codes"].copy())
        base = layout.empty_rows(n, 2 * R, m)
        upper = layout.empty_rows(int(levels.sum()), R, m)
        saved = dict(sm100.BUILD_OPTIONS)
        sm100.BUILD_OPTIONS.update(opts)
        try:
            t0 = time.perf_counter()
            out = sm100.build_graph(4, p, levels, base, uoff, upper, C, R)
            dt = time.perf_counter() - t0
        finally:
            sm100.BUILD_OPTIONS.clear()
            sm100.BUILD_OPTIONS.update(saved)
        graphs[name] = (p, base, upper, out, dt)
    st = search_threads or threads
    res = {}
    for name, (p, base, upper, out, dt) in graphs.items():
        e, ml = out["entry_point"], out["max_layer"]
        r = {"build_s": dt}
        for tag, kind, rr in (("flash", 4, 0), ("rerank64", 4, 64), ("exact", 0, 0)):
            ids, _, _ = core.search_batch(kind, p, levels, base, uoff, upper, C, R, e, ml,
                                          queries, qaux, c["ef"], 10, rr, threads=st,
                                          kernel=kid)
            r[tag] = recall_at_k(ids, gt.ids)
        res[name] = r
    return res


def summarize(per_seed):
    """mean / min / max / per-seed values of every (graph, metric)."""
    out = {}
    for name in per_seed[0]:
        out[name] = {}
        for tag in ("flash", "rerank64", "exact", "build_s"):
            v = np.array([r[name][tag] for r in per_seed])
            out[name][tag] = {"mean": float(v.mean()), "min": float(v.min()),
                              "max": float(v.max()), "values": [float(x) for x in v]}
    return out
