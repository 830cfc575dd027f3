#!/usr/bin/env python
"""One device build of a BASELINE config (for ncu launch lists / captures).

    python scripts/one_build.py [--config 2] [--n N] [--builds 1]

Trains the coder (K9 + K3), projects + encodes (K9 + K2) and runs the default
batched build `--builds` times, nothing else: the launch list of exactly the
bench's hot path.
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2502_18113_b200 import _lib, builder, dataset, flash, graph

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--builds", type=int, default=1)
    ap.add_argument("--hash", action="store_true",
                    help="sha256 of the exported blocks after each build (determinism A/B)")
    ap.add_argument("--profile", action="store_true",
                    help="per-kernel device times (every build after the first)")
    args = ap.parse_args()
    c = dataset.CONFIGS[args.config]
    n = args.n or c["n"]
    x = dataset.baseline_config_dev(args.config, n)
    g0 = torch.Generator(device="cuda").manual_seed(0)
    sample = x[torch.randperm(n, generator=g0, device="cuda")[:100_000].sort().values] \
        if n > 100_000 else x
    model = flash.flash_train(sample, c["d_f"], c["m_f"], seed=0, kmeans_iters=25)
    prov = flash.FlashProvider(model)
    prov.attach(x, vecs_dev=x)
    params = graph.BuildParams(C=c["efC"], R=c["M"], seed=0)
    g = graph.GraphIndex(n, c["dim"], params, "flash", model.m,
                         graph.assign_layers(n, 0, c["M"]))
    g.create_device(prov)
    lib = _lib.load()
    for i in range(args.builds):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        prov.reproject()
        _lib.check(lib.fa_index_set_codes(g.handle, prov.dev["codes"].data_ptr(),
                                          prov.dev["codes"].shape[1], None))
        ctr = builder.build_device(g, prov, params, profile=int(args.profile and i > 0))
        torch.cuda.synchronize()
        ks = "".join(f", {k} {ctr[k]:.2f}" for k in ("ms_encode", "ms_search", "ms_sort", "ms_reverse")
                     if k in ctr)
        ks += "".join(f", {k} {ctr[k]}" for k in ("reverse_prunes", "reverse_full_prunes",
                                                   "reverse_appends") if k in ctr and i == 0)
        print(f"config {args.config} n {n}: {time.perf_counter() - t0:.3f} s, "
              f"{ctr['n_batches']} batches, {ctr['launches']} launches{ks}", flush=True)
        if args.hash:
            import hashlib

            g.invalidate()
            h = hashlib.sha256(g.base_blocks.tobytes())
            h.update(g.upper_blocks.tobytes())
            print("blocks sha256", h.hexdigest()[:16], flush=True)


if __name__ == "__main__":
    main()
