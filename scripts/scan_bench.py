#!/usr/bin/env python
"""Standalone K1 block-scan benchmark for one (m, cap) shape.

    python scripts/scan_bench.py [--m 64 --cap 64] [--reps 5]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=64)
    ap.add_argument("--cap", type=int, default=64)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch

    import bench
    from paper_2502_18113_b200 import _lib

    peak, _ = bench.load_peaks()
    r = bench.scan_benchmark(_lib.load(), torch, args.m, args.cap, peak, reps=args.reps)
    print(json.dumps(r))


if __name__ == "__main__":
    main()
