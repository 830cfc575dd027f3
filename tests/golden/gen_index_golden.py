"""Generate the FANNIDX1 golden file with the REFERENCE package.

Run in the build container (needs /root/reference and `make -C oracle ref`):

    python tests/golden/gen_index_golden.py

The reference trains a Flash coder, builds a 400-vector index with its
compiled core (threads=1, deterministic) and writes it with its own
save_index (flashann/serialize.py:74-113); then the same vectors as an
exact-strategy index.  tests/test_serialize.py reads the
file with this package's reader, re-writes it byte for byte, and (on a GPU)
round-trips it through a device index.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import refpkg  # noqa: E402

OUT = Path(__file__).resolve().parent / "ref_index_small.fannidx"
OUT_EXACT = Path(__file__).resolve().parent / "ref_index_exact.fannidx"


def main() -> None:
    fa = refpkg.import_reference()
    if fa is None:
        raise SystemExit("reference not available (needs /root/reference and oracle/_ref)")
    from flashann import builder, dataset, graph, serialize

    rng = np.random.default_rng(11)
    x = (rng.normal(size=(8, 16))[rng.integers(0, 8, 400)]
         + 0.3 * rng.normal(size=(400, 16))).astype(np.float32)
    ds = dataset.VectorDataset(x)
    res = builder.build(ds, "flash", graph.BuildParams(C=32, R=8, seed=3, threads=1),
                        builder.StrategyParams(m_f=8, d_f=16, kmeans_iters=3))
    serialize.save_index(OUT, res.graph, res.provider, ds)
    print(OUT, OUT.stat().st_size, "bytes")
    # the exact strategy (kind 0): no codes, an empty provider state
    res = builder.build(ds, "exact", graph.BuildParams(C=32, R=8, seed=4, threads=1))
    serialize.save_index(OUT_EXACT, res.graph, res.provider, ds)
    print(OUT_EXACT, OUT_EXACT.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
