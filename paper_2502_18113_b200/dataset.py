"""Datasets, the BASELINE synthetic workloads, and exact k-NN ground truth.

VectorDataset / GroundTruth mirror flashann/dataset.py:19-51.  brute_force_knn
(:126-161: float64 ||q||^2 + ||b||^2 - 2 q.b, clamped, ties by ascending id)
runs on the GPU.  `baseline_config` draws the five BASELINE.json workloads
from seeded generators (no public dataset is named; distributions the
BASELINE text leaves open are the builder's choices documented in DESIGN.md).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._arrays import is_tensor, rows_of
from .errors import ConfigError


@dataclass
class VectorDataset:
    data: np.ndarray  # (n, dim) float32

    def __post_init__(self):
        if not is_tensor(self.data):
            self.data = np.ascontiguousarray(self.data, dtype=np.float32)
        if self.data.ndim != 2:
            raise ConfigError("dataset must be a 2-D array")

    @property
    def n(self) -> int:
        return self.data.shape[0]

    @property
    def dim(self) -> int:
        return self.data.shape[1]

    def __len__(self) -> int:
        return self.n


@dataclass
class GroundTruth:
    k: int
    ids: np.ndarray  # (nq, k) int32
    dists: np.ndarray  # (nq, k) float64


def brute_force_knn(base, queries, k: int, block: int = 256) -> GroundTruth:
    """Exact top-k by squared L2 on the GPU (float64), ties by ascending id."""
    import torch

    b = rows_of(base)
    q = rows_of(queries)
    if b.shape[1] != q.shape[1]:
        raise ConfigError(f"dimension mismatch: base {b.shape[1]} vs queries {q.shape[1]}")
    n = b.shape[0]
    if k > n:
        raise ConfigError(f"k={k} exceeds dataset size {n}")
    bd = torch.as_tensor(b if is_tensor(b) else np.asarray(b), device="cuda").double()
    bsq = (bd * bd).sum(1)
    nq = q.shape[0]
    ids = np.empty((nq, k), np.int32)
    dists = np.empty((nq, k), np.float64)
    qd_all = torch.as_tensor(q if is_tensor(q) else np.asarray(q), device="cuda")
    win = min(n, k + 32)
    ar = torch.arange(n, device="cuda")
    for lo in range(0, nq, block):
        qd = qd_all[lo: lo + block].double()
        d2 = (qd * qd).sum(1)[:, None] + bsq[None, :] - 2.0 * (qd @ bd.T)
        d2.clamp_(min=0.0)
        vals, idx = torch.topk(d2, win, dim=1, largest=False, sorted=True)
        # (d, id) order inside the window: stable sort by id, then by distance
        o = torch.argsort(idx, dim=1, stable=True)
        vals, idx = vals.gather(1, o), idx.gather(1, o)
        o = torch.argsort(vals, dim=1, stable=True)
        vals, idx = vals.gather(1, o), idx.gather(1, o)
        # ties that spill past the window: redo those rows with a full sort
        spill = (vals[:, k - 1] == vals[:, -1]) & (win < n)
        for r in torch.nonzero(spill).flatten().tolist():
            row = d2[r]
            o1 = torch.argsort(ar, stable=True)
            o2 = torch.argsort(row[o1], stable=True)
            idx[r, :] = o1[o2][:win]
            vals[r, :] = row[idx[r]]
        ids[lo: lo + qd.shape[0]] = idx[:, :k].cpu().numpy()
        dists[lo: lo + qd.shape[0]] = vals[:, :k].cpu().numpy()
    return GroundTruth(k=k, ids=ids, dists=dists)


# ---------------------------------------------------------------------------
# BASELINE.json workloads (seeded synthetic stand-ins)

CONFIGS = {
    1: dict(n=20_000, nq=200, dim=128, M=16, efC=100, m_f=32, d_f=128, ef=64),
    2: dict(n=1_000_000, nq=10_000, dim=128, M=32, efC=200, m_f=64, d_f=128, ef=64),
    3: dict(n=10_000_000, nq=10_000, dim=96, M=32, efC=200, m_f=48, d_f=96, ef=64),
    4: dict(n=1_000_000, nq=5_000, dim=960, M=32, efC=300, m_f=64, d_f=256, ef=64),
    5: dict(n=5_000_000, nq=10_000, dim=768, M=48, efC=256, m_f=96, d_f=768, ef=64),
}


def baseline_config(cfg: int, n: int | None = None, nq: int | None = None, seed: int = 0):
    """(base (n, dim) f32, queries (nq, dim) f32) for BASELINE config `cfg`.

    Prefix-stable: the mixture parameters come from one generator and every
    per-row quantity from its own sequential generator, base rows and queries
    on separate streams, so base row i (and query j) is the same for every n
    (nq): a smaller n is exactly the first n rows of the full workload.
    Queries are fresh draws from the same distribution (same mixture
    parameters).  Rows are generated in chunks to bound host memory."""
    c = CONFIGS[cfg]
    n = c["n"] if n is None else n
    nq = c["nq"] if nq is None else nq
    if cfg not in CONFIGS:
        raise ConfigError(f"unknown config {cfg}")
    d = c["dim"]
    prm = np.random.default_rng([seed, cfg, 0])
    if cfg == 1:
        # 64-component isotropic mixture, centres ~ N(0,1), sigma 0.3
        params = dict(centres=prm.normal(0.0, 1.0, (64, d)))
    elif cfg == 2:
        # 256-component mixture, centres ~ U(0,255), sigma 20, rounded, clipped
        params = dict(centres=prm.uniform(0.0, 255.0, (256, d)))
    elif cfg == 3:
        # 1024 components, centres ~ N(0,1), sigma 0.3, then unit L2 norm
        params = dict(centres=prm.normal(0.0, 1.0, (1024, d)))
    elif cfg == 4:
        # 512 components, covariance spectrum i^-1.2 in one random rotation
        q, _ = np.linalg.qr(prm.normal(size=(d, d)))
        params = dict(rot=q, scale=np.arange(1, d + 1, dtype=np.float64) ** -0.6,
                      centres=prm.normal(0.0, 1.0, (512, d)))
    else:
        # rank-64 signal + isotropic noise at SNR 3 (power ratio), unit norm,
        # bf16; the noise power is the signal's expected power / 3
        basis = prm.normal(size=(64, d)) / np.sqrt(d)
        params = dict(basis=basis, noise_sd=np.sqrt((basis ** 2).sum() / d / 3.0))
    return (_rows(cfg, params, n, seed, 1), _rows(cfg, params, nq, seed, 2))


def _rows(cfg: int, p: dict, count: int, seed: int, stream: int, chunk: int = 1 << 18):
    d = CONFIGS[cfg]["dim"]
    ra = np.random.default_rng([seed, cfg, stream, 0])  # component / signal draws
    rn = np.random.default_rng([seed, cfg, stream, 1])  # noise draws
    out = np.empty((count, d), np.float32)
    for lo in range(0, count, chunk):
        s = min(chunk, count - lo)
        if cfg == 1:
            x = p["centres"][ra.integers(0, 64, s)] + rn.normal(0.0, 0.3, (s, d))
        elif cfg == 2:
            x = p["centres"][ra.integers(0, 256, s)] + rn.normal(0.0, 20.0, (s, d))
            x = np.clip(np.rint(x), 0, 255)
        elif cfg == 3:
            x = p["centres"][ra.integers(0, 1024, s)] + rn.normal(0.0, 0.3, (s, d))
            x /= np.linalg.norm(x, axis=1, keepdims=True)
        elif cfg == 4:
            x = p["centres"][ra.integers(0, 512, s)] + (rn.normal(size=(s, d)) * p["scale"]) @ p["rot"].T
        else:
            x = ra.normal(size=(s, 64)) @ p["basis"] + rn.normal(size=(s, d)) * p["noise_sd"]
            x /= np.linalg.norm(x, axis=1, keepdims=True)
            x = _round_bf16(x.astype(np.float32))
        out[lo: lo + s] = x
    return out


def _round_bf16(x: np.ndarray) -> np.ndarray:
    u = x.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


def baseline_config_dev(cfg: int, n: int | None = None, seed: int = 0, chunk: int = 1 << 20):
    """Base rows of BASELINE config `cfg` generated on the GPU (torch, seeded):
    the same law as baseline_config (same mixture / spectrum / rank-64 model,
    the builder's choices of DESIGN §9) from the device RNG, for the bench's
    full-size workloads (10M x 96, 5M x 768) that a host generator would take
    minutes to draw.  Config 5 comes back as bfloat16 (its stated dtype); the
    others as float32.  Not row-identical to baseline_config (another RNG)."""
    import torch

    c = CONFIGS[cfg]
    n = c["n"] if n is None else n
    d = c["dim"]
    g = torch.Generator(device="cuda").manual_seed(1_000_003 * seed + cfg)
    dev = "cuda"
    out = torch.empty((n, d), dtype=torch.bfloat16 if cfg == 5 else torch.float32, device=dev)
    if cfg == 1:
        centres = torch.randn((64, d), generator=g, device=dev)
    elif cfg == 2:
        centres = torch.rand((256, d), generator=g, device=dev) * 255.0
    elif cfg == 3:
        centres = torch.randn((1024, d), generator=g, device=dev)
    elif cfg == 4:
        rot, _ = torch.linalg.qr(torch.randn((d, d), generator=g, device=dev, dtype=torch.float64))
        rot = rot.float()
        scale = torch.arange(1, d + 1, device=dev, dtype=torch.float32) ** -0.6
        centres = torch.randn((512, d), generator=g, device=dev)
    elif cfg == 5:
        basis = torch.randn((64, d), generator=g, device=dev) / (d ** 0.5)
        noise_sd = float(((basis.double() ** 2).sum() / d / 3.0).sqrt())
    else:
        raise ConfigError(f"unknown config {cfg}")
    for lo in range(0, n, chunk):
        s = min(chunk, n - lo)
        if cfg in (1, 2, 3, 4):
            k = centres.shape[0]
            a = torch.randint(0, k, (s,), generator=g, device=dev)
            if cfg == 4:
                x = centres[a] + (torch.randn((s, d), generator=g, device=dev) * scale) @ rot.T
            else:
                sd = {1: 0.3, 2: 20.0, 3: 0.3}[cfg]
                x = centres[a] + torch.randn((s, d), generator=g, device=dev) * sd
            if cfg == 2:
                x = x.round_().clamp_(0, 255)
            if cfg == 3:
                x = x / x.norm(dim=1, keepdim=True)
        else:
            x = torch.randn((s, 64), generator=g, device=dev) @ basis
            x += torch.randn((s, d), generator=g, device=dev) * noise_sd
            x = x / x.norm(dim=1, keepdim=True)
        out[lo: lo + s] = x.to(out.dtype)
    return out
