"""Seeded input generators shared by tests/golden/gen_golden.py and the tests.

Pure numpy; every generator is a fixed function of its seed so the golden
outputs (produced by the reference in the build container) can be checked
anywhere, including the GPU box where /root/reference does not exist.
"""

from __future__ import annotations

import numpy as np

L2_DIMS = list(range(1, 18)) + [24, 31, 32, 33, 64, 96, 128, 768, 960]
SCAN_MS = [1, 8, 16, 24, 32, 48, 64, 96]

MODELS = {
    # name: data shape + coder (dsub = d_f / m_f)
    "t3": {"n": 1500, "dim": 24, "clusters": 8, "d_f": 12, "m_f": 4, "seed": 1, "iters": 25},
    "c1s": {"n": 3000, "dim": 64, "clusters": 16, "d_f": 64, "m_f": 16, "seed": 0, "iters": 10},
    "d2": {"n": 2000, "dim": 64, "clusters": 32, "d_f": 64, "m_f": 32, "seed": 2, "iters": 10},
    "d8": {"n": 2000, "dim": 96, "clusters": 32, "d_f": 64, "m_f": 8, "seed": 3, "iters": 10},
    "mix": {"n": 1200, "dim": 20, "clusters": 4, "d_f": 13, "m_f": 5, "seed": 4, "iters": 5},
}

GRAPH = {"n": 2000, "nq": 100, "dim": 32, "clusters": 24, "sigma": 0.3, "d_f": 32, "m_f": 16,
         "R": 8, "C": 48, "seed": 0, "iters": 10, "ef": 32}
PY_WIDTHS = (4, 16, 48)
# sequential build by the reference's semantic core (_pycore), ~1 min on CPU
PY_BUILD = {"n": 600, "dim": 24, "clusters": 6, "d_f": 24, "m_f": 8, "R": 4, "C": 24, "seed": 5}


def l2_inputs(d: int, count: int = 64):
    rng = np.random.default_rng(1000 + d)
    a = rng.normal(size=(count, d)) * 10.0 ** rng.uniform(-3, 3, size=(count, d))
    b = a + rng.normal(size=(count, d)) * 10.0 ** rng.uniform(-4, 1, size=(count, d))
    return a.astype(np.float32), b.astype(np.float32)


def quantize_inputs():
    rng = np.random.default_rng(7)
    dmin, delta = 0.375, 11.25
    d = rng.uniform(dmin - 0.5 * delta, dmin + 1.5 * delta, 4096)
    d[:6] = (dmin, dmin + delta, dmin + delta / 2, -1.0, 2 * (dmin + delta), np.nextafter(dmin, 0))
    return d, dmin, delta


def scan_cases(m: int, n: int = 30_000, seed: int = 41):
    """Same law as the reference's batch-kernel test (tests/test_flash.py:174-181)."""
    rng = np.random.default_rng(seed + m)
    adts = rng.integers(0, 256, size=(n, m, 16), dtype=np.uint8)
    codes = rng.integers(0, 16, size=(n, m, 16), dtype=np.uint8)
    codes[rng.random(size=codes.shape) < 0.05] = 0
    return adts, codes


def block_case():
    rng = np.random.default_rng(42)
    adt = rng.integers(0, 256, size=(16, 16), dtype=np.uint8)
    flat = rng.integers(0, 16, size=4 * 16 * 16, dtype=np.uint8)
    return adt, flat


def mixture(n, dim, clusters, seed, sigma=1.0, spread=3.0):
    rng = np.random.default_rng(seed)
    centers = rng.normal(0.0, spread, size=(clusters, dim))
    assign = rng.integers(0, clusters, size=n)
    return (centers[assign] + rng.normal(0.0, sigma, size=(n, dim))).astype(np.float32)


def model_data(spec):
    return mixture(spec["n"], spec["dim"], spec["clusters"], 100 + spec["seed"])


def encode_inputs(cent, dims, spec, count: int = 200):
    """Reduced vectors: centroid hits, near-ties between centroids, random."""
    rng = np.random.default_rng(200 + spec["seed"])
    m = cent.shape[0]
    d_f = int(np.sum(dims))
    offs = np.concatenate([[0], np.cumsum(dims)[:-1]]).astype(np.int64)
    red = rng.normal(scale=2.0, size=(count, d_f))
    for r in range(count // 4):  # exact centroid hits
        for i in range(m):
            red[r, offs[i] : offs[i] + dims[i]] = cent[i, rng.integers(16), : dims[i]]
    for r in range(count // 4, count // 2):  # midpoints between two centroids
        for i in range(m):
            a, b = rng.integers(16, size=2)
            red[r, offs[i] : offs[i] + dims[i]] = 0.5 * (cent[i, a, : dims[i]] + cent[i, b, : dims[i]])
    return red.astype(np.float32)


def ulp_inputs(cent, dims, offs, spec, count: int = 120):
    """dist_min/delta such that one uint8 level is ~1 ulp of a real distance."""
    rng = np.random.default_rng(300 + spec["seed"])
    d_f = int(np.sum(dims))
    red = rng.normal(scale=1.5, size=(count, d_f)).astype(np.float32)
    dmins, deltas = np.empty(count), np.empty(count)
    for r in range(count):
        i = int(rng.integers(cent.shape[0]))
        j = int(rng.integers(16))
        x = red[r, offs[i] : offs[i] + dims[i]].astype(np.float64)
        dd = float(np.float32(((x - cent[i, j, : dims[i]]) ** 2).sum()))
        u = float(np.spacing(np.float32(dd)))
        dmins[r] = dd - 100 * u
        deltas[r] = 255 * u
    return red, dmins, deltas


def select_codes(m: int, n: int = 400, seed: int = 11):
    rng = np.random.default_rng(seed)
    # clustered codes so SDT sums tie heavily, as at the BASELINE configs
    base = rng.integers(0, 16, size=(8, m))
    pick = rng.integers(0, 8, size=n)
    codes = base[pick].copy()
    flip = rng.random(size=codes.shape) < 0.25
    codes[flip] = rng.integers(0, 16, size=int(flip.sum()))
    return codes.astype(np.uint8)


def sdt_pairs(codes, count: int = 1000, seed: int = 12):
    rng = np.random.default_rng(seed)
    a = codes[rng.integers(0, codes.shape[0], count)]
    b = codes[rng.integers(0, codes.shape[0], count)]
    return a, b


def select_cases(codes, sdt, count: int = 60, seed: int = 13):
    """(ids, dists, cap): candidate lists sorted by (d, id) like the reference's
    reverse-edge prune (SDT distances to an anchor) and forward prune."""
    rng = np.random.default_rng(seed)
    out = []
    for t in range(count):
        nc = int(rng.integers(2, 120))
        ids = rng.choice(codes.shape[0], size=nc, replace=False).astype(np.int32)
        anchor = codes[int(rng.integers(codes.shape[0]))]
        if t % 2 == 0:  # SDT distances to the anchor (reverse-edge style)
            d = np.array([min(int(sdt[np.arange(len(anchor)), anchor, codes[v]].sum()), 255)
                          for v in ids], dtype=np.float64)
        else:  # small integer ADT-like distances with many ties
            d = rng.integers(0, 6, size=nc).astype(np.float64)
        order = np.lexsort((ids, d))
        cap = int(rng.choice([1, 2, 5, 16, 32, 64]))
        out.append((ids[order], d[order], cap))
    return out


def graph_data():
    g = GRAPH
    allv = mixture(g["n"] + g["nq"], g["dim"], g["clusters"], 500, sigma=g["sigma"], spread=1.0)
    return allv[: g["n"]], allv[g["n"]:]


def flash_narrated():
    """The reference's narrated best-first fixture (tests/util.py:25-48) in
    Flash form: one 2-d subspace whose centroids are the labelled points, so
    every code is exact and the uint8 distances keep the story tie-free.
    Returns (prov, levels, base_blocks (reference layout), uoff, R)."""
    from paper_2502_18113_b200 import layout

    radii = {17: 0.20, 5: 0.30, 3: 0.38, 9: 0.43, 15: 0.47, 0: 0.49, 13: 0.54}
    angles = {17: 0.0, 3: 10.0, 9: -14.0, 5: 95.0, 0: 45.0, 15: -60.0, 13: 150.0}
    pts = np.full((18, 2), 50.0)
    for v, r in radii.items():
        a = np.radians(angles[v])
        pts[v] = (r * np.cos(a), r * np.sin(a))
    labelled = sorted(radii)
    cent = np.zeros((1, 16, 2), np.float32)
    cent[0, : len(labelled)] = pts[labelled]
    cent[0, len(labelled):] = 40.0 + np.arange(16 - len(labelled))[:, None]
    code_of = {v: i for i, v in enumerate(labelled)}
    codes = np.array([[code_of.get(v, 15)] for v in range(18)], np.uint8)
    dmin, delta = 0.0, 0.3
    pair = ((cent[0, :, None, :].astype(np.float64) - cent[0, None, :, :]) ** 2).sum(2)
    t = np.floor((np.clip(pair, dmin, dmin + delta) - dmin) / delta * 255.0)
    sdt = np.where(pair >= dmin + delta, 255, t).astype(np.uint8).reshape(1, 16, 16)
    edges = {0: [5, 9, 13], 5: [0, 15], 9: [0, 17], 17: [9, 3], 3: [17], 15: [5], 13: [0]}
    R = 3
    base = layout.empty_rows(18, 2 * R, 1)
    for v, nb in edges.items():
        layout.set_row(base, v, 2 * R, 1, nb, codes[nb])
    levels = np.zeros(18, np.int32)
    uoff = np.full(18, -1, np.int64)
    prov = {"vecs": pts.astype(np.float32), "dim": 2, "proj": pts.astype(np.float32),
            "codes": codes, "cent": cent, "dims": np.array([2], np.int32),
            "offs": np.array([0], np.int32), "sdt": sdt, "dist_min": dmin, "delta": delta}
    return prov, levels, base, uoff, R
