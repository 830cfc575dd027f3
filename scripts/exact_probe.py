#!/usr/bin/env python
"""Kernel split of a device exact-strategy build (kind 0).

    python scripts/exact_probe.py [--config 2] [--n N]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", type=int, default=None)
    args = ap.parse_args()
    import torch

    from paper_2502_18113_b200 import builder, dataset, graph
    from paper_2502_18113_b200.exact import ExactProvider

    c = dataset.CONFIGS[args.config]
    n = args.n or c["n"]
    data, _ = dataset.baseline_config(args.config, n=n, nq=0)
    prov = ExactProvider()
    prov.attach(data)
    params = graph.BuildParams(C=c["efC"], R=c["M"], seed=0)
    g = graph.GraphIndex(n, data.shape[1], params, "exact", 0, graph.assign_layers(n, 0, c["M"]))
    g.create_device(prov)
    builder.build_device(g, prov, params)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctr = builder.build_device(g, prov, params, profile=1)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"config": args.config, "n": n, "build_s": dt, "vec_per_s": n / dt,
                      "kernel_ms": {k: ctr[k] for k in ("ms_encode", "ms_search", "ms_sort",
                                                         "ms_reverse")},
                      "reverse_prunes": ctr["reverse_prunes"], "n_batches": ctr["n_batches"]}))


if __name__ == "__main__":
    main()
