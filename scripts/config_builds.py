#!/usr/bin/env python
"""Device build throughput at the other BASELINE configs' full sizes.

    python scripts/config_builds.py --configs 3 4 5 [--n N]

For each config: synthetic data of the config's law (dataset.baseline_config),
coder trained on the GPU from a 100K sample, one warm-up build, then one timed
build (re-projection + encode + batched insertion, CUDA events), with the
per-kernel split.  Prints one JSON line per config.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def device_config5(n, seed=0, chunk=1 << 19):
    """Config 5's law (rank-64 signal + isotropic noise at power SNR 3, unit
    norm, bf16-rounded) generated on the device in chunks: 5M x 768 would need
    ~100 GB of float64 host temporaries through dataset.baseline_config."""
    import torch

    d = 768
    g = torch.Generator(device="cuda").manual_seed(seed)
    basis = torch.randn(64, d, device="cuda", generator=g, dtype=torch.float64) / d ** 0.5
    out = torch.empty((n, d), device="cuda", dtype=torch.float32)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        sig = torch.randn(hi - lo, 64, device="cuda", generator=g, dtype=torch.float64) @ basis
        noise = torch.randn(hi - lo, d, device="cuda", generator=g, dtype=torch.float64)
        x = sig + noise * torch.sqrt((sig * sig).mean() / 3.0)
        x /= torch.linalg.norm(x, dim=1, keepdim=True)
        out[lo:hi] = x.to(torch.bfloat16).to(torch.float32)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[3, 4, 5])
    ap.add_argument("--n", type=int, default=None)
    args = ap.parse_args()
    import torch

    from paper_2502_18113_b200 import _lib, builder, dataset, flash, graph

    lib = _lib.load()
    for cfg in args.configs:
        c = dataset.CONFIGS[cfg]
        n = args.n or c["n"]
        t0 = time.perf_counter()
        if cfg == 5 and n > 1_000_000:
            data = x_dev = device_config5(n)
        else:
            data, _ = dataset.baseline_config(cfg, n=n, nq=0)
            x_dev = torch.from_numpy(data).cuda()
        torch.cuda.synchronize()
        gen_s = time.perf_counter() - t0
        sample = builder.training_sample(data, builder.DEFAULT_SAMPLE, 0)
        t0 = time.perf_counter()
        model = flash.flash_train(sample, c["d_f"], c["m_f"], seed=0, kmeans_iters=10)
        torch.cuda.synchronize()
        coding_s = time.perf_counter() - t0
        del sample
        params = graph.BuildParams(C=c["efC"], R=c["M"], seed=0)
        levels = graph.assign_layers(n, 0, c["M"])
        prov = flash.FlashProvider(model)
        prov.attach(data, vecs_dev=x_dev)
        del data
        g = graph.GraphIndex(n, c["dim"], params, "flash", model.m, levels)
        g.create_device(prov)

        def step(profile=0):
            prov.reproject()
            _lib.check(lib.fa_index_set_codes(g.handle, prov.dev["codes"].data_ptr(),
                                              prov.dev["codes"].shape[1], None))
            return builder.build_device(g, prov, params, profile=profile)

        step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctr = step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        prof = step(profile=1)
        print(json.dumps({
            "config": cfg, "n": n, "dim": c["dim"], "m": c["m_f"], "d_f": c["d_f"], "M": c["M"],
            "efConstruction": c["efC"], "vectors_per_s": n / (ms / 1e3), "ms_per_build": ms,
            "kernel_ms": {k: prof[k] for k in ("ms_encode", "ms_search", "ms_sort",
                                                "ms_reverse")},
            "n_batches": ctr["n_batches"], "coding_seconds": coding_s,
            "data_gen_seconds": gen_s}), flush=True)
        g.close()
        del prov, x_dev, g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
