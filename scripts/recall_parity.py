#!/usr/bin/env python
"""Recall@10 parity protocol, run on the GPU box.

Same data, same trained model, two graphs:
  * reference: the reference's own compiled build_graph (oracle/_ref) on the
    host cores (threads=1 is deterministic; threads=all for larger n);
  * sm100: the batched GPU build under the given schedule.
Both graphs are searched by the SAME searcher — the reference's compiled
search_batch — as Flash (ef=64, k=10), Flash + rerank 64, and exact-distance
search on the Flash graph (kind 0 over the same adjacency).  Seeds vary the
layer draws and the training subsample; we report mean and spread.

    python scripts/recall_parity.py --config 1 --seeds 0 1 2 [--threads 1]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import refpkg  # noqa: E402
from paper_2502_18113_b200 import dataset, flash, graph, layout, sm100  # noqa: E402
from paper_2502_18113_b200.evaluation import recall_at_k  # noqa: E402


def build_pair(cfg, n, seed, threads, schedules, ref=True):
    c = dataset.CONFIGS[cfg]
    data, queries = dataset.baseline_config(cfg, n=n, nq=min(c["nq"], 1000))
    gt = dataset.brute_force_knn(data, queries, 10)
    sample = data
    if n > 100_000:
        rng = np.random.default_rng(seed)
        sample = data[np.sort(rng.choice(n, size=100_000, replace=False))]
    model = flash.flash_train(sample, c["d_f"], c["m_f"], seed=seed, kmeans_iters=10)
    prov0 = flash.FlashProvider(model)
    prov0.attach(data)
    pv = prov0.core_arrays()
    qaux = prov0.query_aux(queries)
    R, C = c["M"], c["efC"]
    levels = graph.assign_layers(n, seed, R)
    uoff = graph.upper_offsets_of(levels)
    m = model.m
    core = refpkg.load_ref_core()
    graphs = {}
    if ref:
        p = dict(pv, codes=pv["codes"].copy())
        base = layout.empty_rows(n, 2 * R, m)
        upper = layout.empty_rows(int(levels.sum()), R, m)
        t0 = time.perf_counter()
        out = core.build_graph(4, p, levels, base, uoff, upper, C, R, threads=threads,
                               kernel=len(core.available_kernels()) - 1)
        graphs["reference"] = (p, base, upper, out, time.perf_counter() - t0)
    for name, opts in schedules.items():
        p = dict(pv, codes=pv["codes"].copy())
        base = layout.empty_rows(n, 2 * R, m)
        upper = layout.empty_rows(int(levels.sum()), R, m)
        saved = dict(sm100.BUILD_OPTIONS)
        sm100.BUILD_OPTIONS.update(opts)
        t0 = time.perf_counter()
        out = sm100.build_graph(4, p, levels, base, uoff, upper, C, R)
        dt = time.perf_counter() - t0
        sm100.BUILD_OPTIONS.clear()
        sm100.BUILD_OPTIONS.update(saved)
        graphs[name] = (p, base, upper, out, dt)
    res = {}
    for name, (p, base, upper, out, dt) in graphs.items():
        e, ml = out["entry_point"], out["max_layer"]
        r = {"build_s": dt}
        for tag, kind, rr in (("flash", 4, 0), ("rerank64", 4, 64), ("exact", 0, 0)):
            ids, _, _ = core.search_batch(kind, p, levels, base, uoff, upper, C, R, e, ml,
                                          queries, qaux, 64, 10, rr, threads=16,
                                          kernel=len(core.available_kernels()) - 1)
            r[tag] = recall_at_k(ids, gt)
        res[name] = r
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--seeds", type=int, nargs="+", default=[0, 1, 2])
    ap.add_argument("--threads", type=int, default=1)
    ap.add_argument("--schedules", default="default")
    args = ap.parse_args()
    n = args.n or dataset.CONFIGS[args.config]["n"]
    presets = {
        "seq": dict(batch_max=1, batch_frac=1.0, seq_prefix=1 << 30),
        "f01": dict(batch_max=4096, batch_frac=0.01, seq_prefix=0),
        "f02": dict(batch_max=4096, batch_frac=0.02, seq_prefix=0),
        "f05": dict(batch_max=4096, batch_frac=0.05, seq_prefix=0),
        "f10": dict(batch_max=4096, batch_frac=0.10, seq_prefix=0),
        "f10b16k": dict(batch_max=16384, batch_frac=0.10, seq_prefix=0),
        "f20b64k": dict(batch_max=65536, batch_frac=0.20, seq_prefix=0),
        "f30b64k": dict(batch_max=65536, batch_frac=0.30, seq_prefix=0),
        "default": dict(sm100.BUILD_OPTIONS),
    }
    schedules = {k: presets[k] for k in args.schedules.split(",")}
    allres = []
    for s in args.seeds:
        r = build_pair(args.config, n, s, args.threads, schedules)
        allres.append(r)
        print(json.dumps({"seed": s, **r}), flush=True)
    summary = {}
    for name in allres[0]:
        summary[name] = {}
        for tag in ("flash", "rerank64", "exact", "build_s"):
            v = np.array([r[name][tag] for r in allres])
            summary[name][tag] = {"mean": float(v.mean()), "min": float(v.min()),
                                  "max": float(v.max())}
    print(json.dumps({"config": args.config, "n": n, "seeds": args.seeds,
                      "ref_threads": args.threads, "summary": summary}))


if __name__ == "__main__":
    main()
