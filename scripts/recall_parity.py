#!/usr/bin/env python
"""Recall@10 parity protocol, run on the GPU box.

    python scripts/recall_parity.py --config 2 [--n 1000000] [--seeds 0 1 2]
                                    [--threads 16] [--nq 10000] [--out f.json]

oracle/recall.py: same data and coder, the reference's compiled build_graph
(host cores) vs the default batched GPU build, both searched by the
reference's compiled search_batch (Flash ef 64, Flash + rerank 64, exact
search over the graph).  Configs 3 and 5 run on 1M-vector prefixes of the
(prefix-stable) synthetic workload: the CPU reference cannot build 10M / 5M
in-run.  Prints one JSON line per seed and a summary with per-seed values.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import recall  # noqa: E402
from paper_2502_18113_b200 import dataset  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--nq", type=int, default=None)
    ap.add_argument("--seeds", type=int, nargs="+", default=[0, 1, 2])
    ap.add_argument("--threads", type=int, default=1)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    c = dataset.CONFIGS[args.config]
    n = args.n or min(c["n"], 1_000_000)
    nq = args.nq or c["nq"]
    t0 = time.time()
    data, queries = dataset.baseline_config(args.config, n=n, nq=nq)
    print(json.dumps({"generated_s": time.time() - t0, "n": n, "nq": nq}), flush=True)
    per_seed = []
    for s in args.seeds:
        r = recall.build_pair(args.config, n, nq, s, threads=args.threads,
                              search_threads=args.threads, data=data, queries=queries)
        per_seed.append(r)
        print(json.dumps({"seed": s, **r}), flush=True)
    summary = {"config": args.config, "n": n, "n_full": c["n"], "nq": nq, "seeds": args.seeds,
               "ref_threads": args.threads,
               "prefix": n < c["n"],
               "protocol": "oracle/recall.py: same data + coder; reference compiled build_graph "
                           "vs default GPU build; both searched by the reference's compiled "
                           f"search_batch, ef {c['ef']}, k 10",
               "summary": recall.summarize(per_seed)}
    print(json.dumps(summary), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(summary, indent=1) + "\n")


if __name__ == "__main__":
    main()
