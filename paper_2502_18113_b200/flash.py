"""Flash coder on the GPU: rotation, 16-centroid subspace codebooks, the shared
uint8 distance grid, the symmetric table, and the bulk encoder.

Mirrors flashann/flash.py (FlashModel :32-49, quantize_distance :52-56,
flash_train :63-107, encode_and_adt :110-115, sdt_distance :118-123,
FlashProvider :141-227).  Training runs K3 (csrc/kmeans.cu) for every
subspace at once; the random stream is numpy's PCG64 continued on the device
from the host-drawn subsample permutation, so the draws are the reference's.
Encoding runs K2 (csrc/encode.cu) with the compiled core's fp32 operation tree
— i.e. the codes the reference's build leaves in prov["codes"]
(_core.pyx:493-498), not the float64 expansion of its bulk pre-encode.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from ._arrays import rows_of
from ._lib import check
from .errors import ConfigError
from .pca import PCAModel, as_device_f32, pca_project, pca_project_all_dev, pca_train

K = 16
QMAX = 255
MAX_POINTS_PER_CENTROID = 256  # kmeans.py:13


@dataclass
class FlashModel:
    pca: PCAModel
    m: int
    dims: np.ndarray  # (m,) int32
    offs: np.ndarray  # (m,) int32
    cent: np.ndarray  # (m, 16, dmax) float32, zero padded
    sdt: np.ndarray  # (m, 16, 16) uint8
    dist_min: float
    dist_max: float

    @property
    def delta(self) -> float:
        return self.dist_max - self.dist_min

    @property
    def d(self) -> int:
        return self.pca.d


def split_dims(dim: int, m: int):
    """ceil widths for the first dim % m subspaces, then floor (pq.py:20-28)."""
    if m < 1 or m > dim:
        raise ConfigError(f"subspace count {m} invalid for dimension {dim}")
    q, r = divmod(dim, m)
    sizes = np.array([q + 1] * r + [q] * (m - r), dtype=np.int32)
    offs = np.zeros(m, dtype=np.int32)
    offs[1:] = np.cumsum(sizes)[:-1]
    return sizes, offs


def _torch():
    import torch

    return torch


def _lib_():
    return _lib.load()


def quantize_distance(model: FlashModel, dist) -> np.ndarray:
    if model.delta <= 0:
        raise ConfigError("degenerate quantization range")
    from . import sm100

    return sm100.quantize_distance(dist, model.dist_min, model.delta)


def dequantize_distance(model: FlashModel, q) -> np.ndarray:
    return model.dist_min + np.asarray(q, dtype=np.float64) * model.delta / QMAX


_PCG_DT = np.dtype([("s_hi", "<u8"), ("s_lo", "<u8"), ("inc_hi", "<u8"), ("inc_lo", "<u8"),
                    ("has", "<u4"), ("u", "<u4")])


def _rng_streams(ns: int, m: int, seed: int):
    """Per-subspace subsample rows and the PCG64 state after drawing them
    (kmeans.py:50-54: default_rng(seed+i); permutation(n)[:k*256], sorted).
    The permutations run in the core library on the host cores
    (fa_kmeans_subsample); numpy only seeds the generators."""
    cap = K * MAX_POINTS_PER_CENTROID
    states = np.zeros(m, dtype=_PCG_DT)
    for i in range(m):
        st = np.random.default_rng(seed + i).bit_generator.state
        s, inc = st["state"]["state"], st["state"]["inc"]
        states[i] = (s >> 64, s & ((1 << 64) - 1), inc >> 64, inc & ((1 << 64) - 1),
                     st["has_uint32"], st["uinteger"])
    if ns <= cap:
        return None, states
    sel = np.zeros((m, cap), dtype=np.int32)
    check(_lib.load(require_device=False).fa_kmeans_subsample(
        ns, cap, m, states.ctypes.data, sel.ctypes.data))
    return sel, states


def train_codebooks(reduced, dims, offs, seed: int = 0, kmeans_iters: int = 25):
    """K3 on the device for all subspaces of the reduced sample.

    Returns (cent (m,16,dmax) f32, sdt (m,16,16) u8, dist_min, dist_max,
    history (m, iters+1) f64)."""
    torch = _torch()
    lib = _lib_()
    x = as_device_f32(reduced)
    ns, dF = x.shape
    dims = np.ascontiguousarray(dims, np.int32)
    offs = np.ascontiguousarray(offs, np.int32)
    m = dims.shape[0]
    dmax = int(dims.max())
    if ns < K:
        raise ValueError(f"need at least {K} training points, got {ns}")
    sel, states = _rng_streams(ns, m, seed)
    nsub = sel.shape[1] if sel is not None else ns
    d_dims = torch.from_numpy(dims).cuda()
    d_offs = torch.from_numpy(offs).cuda()
    d_sel = torch.from_numpy(sel).cuda() if sel is not None else None
    d_states = torch.from_numpy(states.view(np.uint8)).cuda()
    scratch = torch.empty(int(lib.fa_kmeans_scratch_bytes(m, nsub)), dtype=torch.uint8,
                          device="cuda")
    cent = torch.zeros((m, K, dmax), dtype=torch.float32, device="cuda")
    hist = torch.zeros((m, kmeans_iters + 1), dtype=torch.float64, device="cuda")
    check(lib.fa_kmeans_subspaces_dev(
        x.data_ptr(), ns, dF, d_dims.data_ptr(), d_offs.data_ptr(), m,
        d_sel.data_ptr() if d_sel is not None else None, nsub, d_states.data_ptr(),
        int(kmeans_iters), cent.data_ptr(), dmax, hist.data_ptr(), scratch.data_ptr(), None))
    raw = torch.empty((m, K, K), dtype=torch.float64, device="cuda")
    rng_out = torch.empty(2, dtype=torch.float64, device="cuda")
    scr2 = torch.empty(3 * m + 8, dtype=torch.float64, device="cuda")
    check(lib.fa_flash_range_dev(x.data_ptr(), ns, dF, d_dims.data_ptr(), d_offs.data_ptr(), m,
                                 cent.data_ptr(), dmax, raw.data_ptr(), rng_out.data_ptr(),
                                 scr2.data_ptr(), None))
    dist_min, dist_max = (float(v) for v in rng_out.cpu().numpy())
    if dist_max <= dist_min:
        raise ConfigError("degenerate sample: zero distance spread")
    sdt = torch.empty((m, K, K), dtype=torch.uint8, device="cuda")
    check(lib.fa_quantize_dev(raw.data_ptr(), m * K * K, dist_min, dist_max - dist_min,
                              sdt.data_ptr(), None))
    return (cent.cpu().numpy(), sdt.cpu().numpy(), dist_min, dist_max, hist.cpu().numpy())


def flash_train(sample, d_f: int, m_f: int, seed: int = 0, kmeans_iters: int = 25) -> FlashModel:
    """Fit rotation, codebooks, quantization range and the symmetric table
    (flash.py:63-107) on the GPU."""
    data = rows_of(sample)
    n, dim = data.shape
    if n < 10 * K:
        raise ConfigError(f"need at least {10 * K} training vectors, got {n}")
    if not 1 <= d_f <= dim:
        raise ConfigError(f"d_f={d_f} out of range for dimension {dim}")
    if m_f > d_f:
        raise ConfigError(f"m_f={m_f} exceeds projection width {d_f}")
    pca = pca_train(sample, d=d_f)
    reduced = pca_project_all_dev(pca, data)
    dims, offs = split_dims(d_f, m_f)
    cent, sdt, dmin, dmax, _ = train_codebooks(reduced, dims, offs, seed, kmeans_iters)
    return FlashModel(pca=pca, m=m_f, dims=dims, offs=offs, cent=cent, sdt=sdt,
                      dist_min=dmin, dist_max=dmax)


def encode_rows_dev(model: FlashModel, proj_dev, code_stride: int | None = None):
    """Codes (n, code_stride) u8 on the device for projected rows (K2)."""
    torch = _torch()
    lib = _lib_()
    n = proj_dev.shape[0]
    cs = model.m if code_stride is None else code_stride
    codes = torch.zeros((n, cs), dtype=torch.uint8, device="cuda")
    dm = _model_dev(model)
    if n:
        check(lib.fa_encode_adt_dev(proj_dev.data_ptr(), n, proj_dev.shape[1],
                                    dm["cent"].data_ptr(), dm["dims"].data_ptr(),
                                    dm["offs"].data_ptr(), model.m, model.cent.shape[2],
                                    model.dist_min, model.delta, codes.data_ptr(), cs, None, 0,
                                    None))
    return codes


def _model_dev(model: FlashModel) -> dict:
    cache = getattr(model, "_dev_cache", None)
    if cache is None:
        torch = _torch()
        cache = {
            "cent": torch.from_numpy(np.ascontiguousarray(model.cent, np.float32)).cuda(),
            "dims": torch.from_numpy(np.ascontiguousarray(model.dims, np.int32)).cuda(),
            "offs": torch.from_numpy(np.ascontiguousarray(model.offs, np.int32)).cuda(),
            "sdt": torch.from_numpy(np.ascontiguousarray(model.sdt, np.uint8)).cuda(),
        }
        model._dev_cache = cache
    return cache


def encode_and_adt(model: FlashModel, vec):
    """Codewords and quantized query table of one vector (flash.py:110-115)."""
    from . import sm100

    red = pca_project(model.pca, vec).astype(np.float32)
    return sm100.flash_encode_adt(model.cent, model.dims, model.offs, model.dist_min,
                                  model.delta, red)


def sdt_distance(model: FlashModel, code_a, code_b) -> int:
    for c in (code_a, code_b):
        if np.any(np.asarray(c) >= K):
            raise ConfigError("codeword value out of range")
    from . import sm100

    return sm100.flash_sdt_distance(model.sdt, np.asarray(code_a), np.asarray(code_b))


class FlashProvider:
    """Flash strategy bound to one dataset; arrays stay resident on the GPU.

    core_arrays() returns the reference's host `prov` dict
    (flash.py:157-168) for the core-module drop-in path."""

    kind = "flash"
    kind_id = 4

    def __init__(self, model: FlashModel):
        self.model = model
        self.dataset = None
        self.dev: dict = {}
        self._prov = None

    @property
    def code_subspaces(self) -> int:
        return self.model.m

    def attach(self, dataset, vecs_dev=None) -> None:
        """Project + encode every row on the device."""
        data = rows_of(dataset)
        if data.shape[1] != self.model.pca.mean.shape[0]:
            raise ConfigError("dataset dimension does not match the trained model")
        self.dataset = dataset
        x = vecs_dev if vecs_dev is not None else as_device_f32(data)
        proj = pca_project_all_dev(self.model.pca, x)
        mpad = -(-self.model.m // 16) * 16
        codes = encode_rows_dev(self.model, proj, mpad)
        self.dev = {"vecs": x, "proj": proj, "codes": codes, **_model_dev(self.model)}
        self._prov = None

    def reproject(self, lo: int = 0, hi: int | None = None) -> None:
        """Recompute projection + codes of the attached rows [lo, hi) in place
        (the device buffers keep their addresses, so a device index stays
        valid)."""
        hi = self.dev["codes"].shape[0] if hi is None else hi
        if hi <= lo:
            return
        proj = pca_project_all_dev(self.model.pca, self.dev["vecs"][lo:hi])
        self.dev["proj"][lo:hi].copy_(proj)
        del proj
        lib = _lib_()
        dm = _model_dev(self.model)
        codes = self.dev["codes"]
        pr = self.dev["proj"]
        check(lib.fa_encode_adt_dev(pr[lo].data_ptr(), hi - lo, pr.shape[1],
                                    dm["cent"].data_ptr(), dm["dims"].data_ptr(),
                                    dm["offs"].data_ptr(), self.model.m,
                                    self.model.cent.shape[2], self.model.dist_min,
                                    self.model.delta, codes[lo].data_ptr(), codes.shape[1],
                                    None, 0, None))
        self._prov = None

    def core_arrays(self) -> dict:
        if not self.dev:
            raise ConfigError("provider not attached to a dataset")
        if self._prov is None:
            data = rows_of(self.dataset)
            self._prov = {
                "vecs": data if isinstance(data, np.ndarray) else self.dev["vecs"].cpu().numpy(),
                "dim": int(self.dev["vecs"].shape[1]),
                "proj": self.dev["proj"].cpu().numpy(),
                "codes": np.ascontiguousarray(self.dev["codes"][:, : self.model.m].cpu().numpy()),
                "cent": self.model.cent, "dims": self.model.dims, "offs": self.model.offs,
                "sdt": self.model.sdt, "dist_min": self.model.dist_min,
                "delta": self.model.delta,
            }
        return self._prov

    def encode(self, vec):
        return encode_and_adt(self.model, vec)[0]

    def query_aux(self, queries) -> np.ndarray:
        return pca_project_all_dev(self.model.pca, queries).cpu().numpy()

    def query_aux_dev(self, queries_dev):
        return pca_project_all_dev(self.model.pca, queries_dev)

    def sym_distance(self, a: int, b: int) -> float:
        codes = self.dev["codes"]
        return float(sdt_distance(self.model, codes[a, : self.model.m].cpu().numpy(),
                                  codes[b, : self.model.m].cpu().numpy()))

    def state_dict(self) -> dict:
        p = self.model.pca
        return {"mean": p.mean, "basis": p.basis, "eigvals": p.eigvals, "d": p.d,
                "m": self.model.m, "dims": self.model.dims, "offs": self.model.offs,
                "cent": self.model.cent, "sdt": self.model.sdt,
                "dist_min": self.model.dist_min, "dist_max": self.model.dist_max}

    @classmethod
    def from_state(cls, state: dict) -> "FlashProvider":
        pca = PCAModel(mean=state["mean"], basis=state["basis"], eigvals=state["eigvals"],
                       d=int(state["d"]))
        return cls(FlashModel(pca=pca, m=int(state["m"]), dims=state["dims"], offs=state["offs"],
                              cent=state["cent"], sdt=state["sdt"],
                              dist_min=float(state["dist_min"]),
                              dist_max=float(state["dist_max"])))

