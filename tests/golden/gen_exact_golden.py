"""Golden fixtures for the EXACT strategy (kind 0) from the REFERENCE package.

Run in the build container (needs /root/reference and `make -C oracle ref`):

    python tests/golden/gen_exact_golden.py

The reference's semantic core (_pycore: heap rules, ties by vertex id) builds
and searches an exact-strategy graph with the compiled core's fp32 distance
(fa_l2sq_f32, _core.pyx:167-191 asym_one / sym_one for K_EXACT) substituted
for _pycore's float64 sums — the same substitution the Flash golden build makes
for the encoder.  Sequential insertion, so the oracle's exact build at batch
size 1 must reproduce it row for row.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle import refpkg  # noqa: E402
import golden_inputs as gi  # noqa: E402

OUT = Path(__file__).resolve().parent / "exact_golden.npz"
EX = {"n": 500, "dim": 20, "clusters": 6, "R": 4, "C": 20, "seed": 7, "nq": 40, "ef": 24, "k": 8}


def main() -> None:
    fa = refpkg.import_reference()
    if fa is None:
        raise SystemExit("reference not available (needs /root/reference and oracle/_ref)")
    EXT = fa.core.impl
    pyc = fa._pycore
    orig_asym, orig_sym = pyc._Dist.asym_many, pyc._Dist.sym_many

    def asym_many(self, ctx, ids):
        if self.kind != 0:
            return orig_asym(self, ctx, ids)
        q = np.asarray(ctx["vec"], np.float32)
        return np.array([EXT.l2sq_f32(q, self.p["vecs"][int(i)]) for i in ids], np.float64)

    def sym_many(self, v, ids):
        if self.kind != 0:
            return orig_sym(self, v, ids)
        a = self.p["vecs"][int(v)]
        return np.array([EXT.l2sq_f32(a, self.p["vecs"][int(i)]) for i in ids], np.float64)

    pyc._Dist.asym_many, pyc._Dist.sym_many = asym_many, sym_many
    try:
        data = gi.mixture(EX["n"] + EX["nq"], EX["dim"], EX["clusters"], 4242, sigma=0.5,
                          spread=1.0)
        base_x, queries = data[: EX["n"]], data[EX["n"]:]
        prov = {"vecs": base_x, "dim": EX["dim"]}
        levels = fa.assign_layers(EX["n"], EX["seed"], EX["R"])
        g = fa.GraphIndex(EX["n"], EX["dim"], fa.BuildParams(C=EX["C"], R=EX["R"]), "exact", 0,
                          levels)
        res = pyc.build_graph(0, prov, levels, g.base_blocks, g.upper_offsets, g.upper_blocks,
                              EX["C"], EX["R"])
        ids, ds, _ = pyc.search_batch(0, prov, levels, g.base_blocks, g.upper_offsets,
                                      g.upper_blocks, EX["C"], EX["R"], res["entry_point"],
                                      res["max_layer"], queries, None, EX["ef"], EX["k"], 0)
    finally:
        pyc._Dist.asym_many, pyc._Dist.sym_many = orig_asym, orig_sym
    np.savez_compressed(OUT, vecs=base_x, queries=queries, levels=levels,
                        uoff=g.upper_offsets, base=g.base_blocks, upper=g.upper_blocks,
                        state=np.array([res["entry_point"], res["max_layer"]]), ids=ids, d=ds,
                        params=np.array([EX["R"], EX["C"], EX["ef"], EX["k"]]))
    print("wrote", OUT, res["entry_point"], res["max_layer"], res["counters"])


if __name__ == "__main__":
    main()
