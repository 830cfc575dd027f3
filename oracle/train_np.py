"""numpy restatement of the reference coder training (TEST/BASELINE ONLY).

Follows flashann/providers/pca.py:27-71 (pca_train / pca_project_all),
flashann/kmeans.py:16-76 (k-means++ + Lloyd, float64, PCG64 draws),
flashann/flash.py:63-107 (range + SDT) and flashann/builder.py:60-65
(training sample).  Used as the checker for the GPU trainer and as the CPU
training step of bench.py's reference arm on the GPU box (where the
reference's own Python is absent).  Pinned against the reference's golden
models in tests/test_oracle_train.py.
"""

from __future__ import annotations

import numpy as np

K = 16
CAP = 16 * 256


def pca(data: np.ndarray, d: int):
    x = data.astype(np.float64)
    mean = x.mean(0)
    xc = (data - mean.astype(np.float32)).astype(np.float32)
    cov = (xc.T @ xc).astype(np.float64) / data.shape[0]
    w, v = np.linalg.eigh(cov)
    return mean, v[:, ::-1].copy(), np.maximum(w[::-1], 0.0), d


def project(mean, basis, d, data):
    return ((data.astype(np.float32) - mean.astype(np.float32))
            @ basis[:, :d].astype(np.float32)).astype(np.float32)


def _seed_plusplus(x, rng):
    n = x.shape[0]
    c = np.empty((K, x.shape[1]))
    c[0] = x[int(rng.integers(n))]
    d2 = ((x - c[0]) ** 2).sum(1)
    for j in range(1, K):
        tot = d2.sum()
        if tot <= 0:
            c[j] = x[int(rng.integers(n))]
            continue
        r = rng.random() * tot
        c[j] = x[min(int(np.searchsorted(np.cumsum(d2), r)), n - 1)]
        d2 = np.minimum(d2, ((x - c[j]) ** 2).sum(1))
    return c


def kmeans(sub: np.ndarray, iters: int, seed: int):
    x = np.asarray(sub, dtype=np.float64)
    rng = np.random.default_rng(seed)
    if x.shape[0] > CAP:
        x = x[np.sort(rng.permutation(x.shape[0])[:CAP])]
    n = x.shape[0]
    c = _seed_plusplus(x, rng)
    xsq = (x * x).sum(1)
    hist = np.empty(iters + 1)
    for it in range(iters + 1):
        d2 = xsq[:, None] + (c * c).sum(1)[None, :] - 2.0 * (x @ c.T)
        a = d2.argmin(1)
        best = np.maximum(d2[np.arange(n), a], 0.0)
        hist[it] = best.sum()
        if it == iters:
            break
        cnt = np.bincount(a, minlength=K)
        s = np.zeros_like(c)
        np.add.at(s, a, x)
        ok = cnt > 0
        c[ok] = s[ok] / cnt[ok, None]
        for j in np.flatnonzero(~ok):
            far = int(best.argmax())
            c[j] = x[far]
            best[far] = 0.0
    return c.astype(np.float32), hist


def split_dims(d: int, m: int):
    q, r = divmod(d, m)
    dims = np.array([q + 1] * r + [q] * (m - r), np.int32)
    offs = np.concatenate([[0], np.cumsum(dims)[:-1]]).astype(np.int32)
    return dims, offs


def quantize(d, dmin, delta):
    d = np.asarray(d, np.float64)
    top = dmin + delta
    t = np.clip(np.floor((np.clip(d, dmin, top) - dmin) / delta * 255.0), 0.0, 255.0)
    return np.where(d >= top, 255.0, t).astype(np.uint8)


def train(data: np.ndarray, d_f: int, m_f: int, seed: int = 0, iters: int = 25):
    """-> dict(mean, basis, d, dims, offs, cent, sdt, dist_min, dist_max)."""
    mean, basis, eig, d = pca(data, d_f)
    red = project(mean, basis, d, data)
    dims, offs = split_dims(d_f, m_f)
    cent = np.zeros((m_f, K, int(dims.max())), np.float32)
    raw = np.empty((m_f, K, K))
    lo, hi = np.empty(m_f), np.empty(m_f)
    for i in range(m_f):
        sub = red[:, offs[i]: offs[i] + dims[i]]
        c, _ = kmeans(sub, iters, seed + i)
        cent[i, :, : dims[i]] = c
        c64 = c.astype(np.float64)
        pair = ((c64[:, None, :] - c64[None, :, :]) ** 2).sum(2)
        raw[i] = pair
        s64 = sub.astype(np.float64)
        x2 = np.maximum((s64 * s64).sum(1)[:, None] + (c64 * c64).sum(1)[None, :]
                        - 2.0 * (s64 @ c64.T), 0.0)
        lo[i] = min(pair.min(), x2.min())
        hi[i] = max(pair.max(), x2.max())
    dmin, dmax = float(lo.min()), float(hi.sum())
    return {"mean": mean, "basis": basis, "eigvals": eig, "d": d, "dims": dims, "offs": offs,
            "cent": cent, "sdt": quantize(raw, dmin, dmax - dmin), "dist_min": dmin,
            "dist_max": dmax, "proj_fn": lambda x: project(mean, basis, d, x)}


def training_sample(data: np.ndarray, size: int, seed: int) -> np.ndarray:
    if data.shape[0] <= size:
        return data
    rng = np.random.default_rng(seed)
    return data[np.sort(rng.choice(data.shape[0], size=size, replace=False))]
