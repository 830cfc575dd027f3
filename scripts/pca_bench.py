#!/usr/bin/env python
"""K9 timing: the PCA covariance and projection GEMMs at the BASELINE shapes.

    python scripts/pca_bench.py [--out profiles/rNN_pca_gemm.json]

c4: covariance of the 100K training sample (960 x 960), projection of 1M rows
960 -> 256; c5: covariance of 100K bf16 rows (768 x 768), projection of 5M
bf16 rows 768 -> 768.  Device-resident inputs, CUDA events, 3xTF32 (3 MMAs
per product): "tflops" counts the useful 2*n*D*d flops, "tc_tflops" the
tensor-core flops issued (x3), against MEASURED_PEAKS' dense bf16 peak / 2
(tf32 runs at half the bf16 rate).
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np
    import torch

    from paper_2502_18113_b200 import pca

    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    bf16_peak = float(peaks.get("bf16_tflops", peaks.get("dense_bf16_tflops", 2250.0)))
    g = torch.Generator(device="cuda").manual_seed(0)
    res = {}

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    for name, n, D, d, dt, ncov in (("c4", 1_000_000, 960, 256, torch.float32, 100_000),
                                     ("c5", 5_000_000, 768, 768, torch.bfloat16, 100_000)):
        x = torch.randn((n, D), generator=g, device="cuda", dtype=torch.float32).to(dt)
        mean = x[:ncov].double().mean(0).float().contiguous()
        q, _ = torch.linalg.qr(torch.randn((D, D), generator=g, device="cuda", dtype=torch.float64))
        model = pca.PCAModel(mean=mean.double().cpu().numpy(), basis=q.cpu().numpy(),
                             eigvals=np.ones(D), d=d)
        ms_cov = timed(lambda: pca.covariance_dev(x[:ncov], mean))
        ms_proj = timed(lambda: pca.pca_project_all_dev(model, x), reps=3)
        fl_cov = 2.0 * ncov * D * D / 2  # upper triangle of tiles (about half)
        fl_proj = 2.0 * n * D * d
        res[name] = {
            "dtype": str(dt).replace("torch.", ""),
            "cov": {"n": ncov, "D": D, "ms": ms_cov, "tflops": fl_cov / ms_cov / 1e9,
                    "tc_tflops": 3 * fl_cov / ms_cov / 1e9},
            "proj": {"n": n, "D": D, "d": d, "ms": ms_proj, "tflops": fl_proj / ms_proj / 1e9,
                     "tc_tflops": 3 * fl_proj / ms_proj / 1e9,
                     "hbm_gbs": x.element_size() * n * D / ms_proj / 1e6},
        }
        del x
        torch.cuda.empty_cache()
    out = {"tf32_dense_peak_tflops": bf16_peak / 2, "peak_basis": "MEASURED_PEAKS bf16 / 2",
           **res}
    print(json.dumps(out))
    if args.out:
        Path(args.out).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
