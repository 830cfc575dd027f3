#!/usr/bin/env python
"""Diagnostics of one device build: per-kernel time, batch count and the
distribution of per-insertion search work (expansions, SM cycles).

    python scripts/probe_build.py --config 2 --n 200000 [--frac 0.1] [--bmax 4096]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2502_18113_b200 import builder, dataset, flash, graph, sm100  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", type=int, default=200_000)
    ap.add_argument("--frac", type=float, default=None)
    ap.add_argument("--bmax", type=int, default=None)
    ap.add_argument("--hash-log2", type=int, default=0)
    ap.add_argument("--tie", type=int, default=None)
    ap.add_argument("--expand", type=int, default=None)
    ap.add_argument("--dump", default=None, help="save the per-point stats (.npy)")
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    import torch

    c = dataset.CONFIGS[args.config]
    data, _ = dataset.baseline_config(args.config, n=args.n, nq=0)
    model = flash.flash_train(builder.training_sample(data, 100_000, 0), c["d_f"], c["m_f"], 0, 10)
    prov = flash.FlashProvider(model)
    prov.attach(data)
    params = graph.BuildParams(C=c["efC"], R=c["M"], seed=0)
    g = graph.GraphIndex(args.n, data.shape[1], params, "flash", model.m,
                         graph.assign_layers(args.n, 0, c["M"]))
    g.create_device(prov)
    over = {"hash_log2": args.hash_log2}
    if args.frac is not None:
        over["batch_frac"] = args.frac
    if args.bmax is not None:
        over["batch_max"] = args.bmax
    if args.tie is not None:
        over["tie"] = args.tie
    if args.expand is not None:
        over["expand"] = args.expand
    stats = torch.zeros((args.n, 8), dtype=torch.int64, device="cuda")
    for r in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctr = builder.build_device(g, prov, params, profile=1, **over)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    # one more with per-point stats
    from paper_2502_18113_b200 import _lib
    import ctypes as C

    opts = builder.build_options(params, profile=0, **over)
    opts.point_stats = stats.data_ptr()
    res = _lib.BuildResult()
    _lib.check(_lib.load().fa_index_build(g.handle, C.byref(opts), C.byref(res), None))
    st = stats.cpu().numpy()[1:]
    if args.dump:
        np.save(args.dump, stats.cpu().numpy())
    exp, cyc = st[:, 0], st[:, 1]
    q = [50, 90, 99, 99.9, 100]
    print(json.dumps({
        "n": args.n, "build_s": dt, "vec_per_s": args.n / dt, "options": over,
        "kernel_ms": {k: ctr[k] for k in ("ms_encode", "ms_search", "ms_sort", "ms_reverse")},
        "n_batches": ctr["n_batches"], "reverse_prunes": ctr["reverse_prunes"],
        "reverse_full_prunes": ctr["reverse_full_prunes"],
        "expansions": {"mean": float(exp.mean()), **{f"p{p}": float(np.percentile(exp, p))
                                                     for p in q}},
        "kcycles": {"mean": float(cyc.mean() / 1e3), **{f"p{p}": float(np.percentile(cyc, p) / 1e3)
                                                        for p in q}},
        "cycles_per_expansion": float(cyc.sum() / max(exp.sum(), 1)),
        "phase_cycles_per_expansion": {
            name: float(st[:, 2 + i].sum() / max(exp.sum(), 1))
            for i, name in enumerate(["pop", "row_visit", "dists", "accept"])},
        "select_cycles_per_insert": float(st[:, 6].mean()),
        "dist_per_expansion": float(st[:, 7].sum() / max(exp.sum(), 1)),
    }))


if __name__ == "__main__":
    main()
