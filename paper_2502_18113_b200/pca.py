"""Rotation used by the Flash coder (flashann/providers/pca.py:27-71), on the GPU.

pca_train: float64 mean, the float32-centred covariance as a 3xTF32 tcgen05
GEMM (K9, csrc/pca_gemm.cu; the reference's fp32 sgemm, pca.py:36-38),
float64 symmetric eigendecomposition (cuSOLVER), components by descending
eigenvalue, eigenvalues clamped at 0.
pca_project_all: (x - mean) @ basis[:, :d] as a 3xTF32 tcgen05 GEMM fed by
TMA (pca.py:68-71), rows in float32 or bfloat16 (bf16 is widened exactly).
pca_project: the reference's float64 single-vector projection (pca.py:57-65).

Eigenvectors are defined up to sign (and up to rotation inside degenerate
eigenspaces); everything downstream (codes, tables, the graph) is invariant
to a per-component sign, and parity tests compare bases up to sign.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from ._arrays import is_tensor, rows_of
from ._lib import check
from .errors import ConfigError


@dataclass
class PCAModel:
    mean: np.ndarray  # (dim,) float64
    basis: np.ndarray  # (dim, dim) float64, columns by descending eigenvalue
    eigvals: np.ndarray  # (dim,) float64, non-increasing
    d: int


def _torch():
    import torch

    if not torch.cuda.is_available():
        from .errors import DeviceError

        raise DeviceError("no CUDA device visible: training runs on the GPU only")
    return torch


def as_device_f32(data):
    torch = _torch()
    if is_tensor(data):
        return data.to(device="cuda", dtype=torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(data, dtype=np.float32)).cuda()


def as_device_rows(data):
    """Rows on the device in float32, or bfloat16 when given as a bf16 tensor
    (the tensor-core contractions widen bf16 exactly; half the bytes)."""
    torch = _torch()
    if is_tensor(data) and data.dtype == torch.bfloat16:
        return data.to(device="cuda").contiguous()
    return as_device_f32(data)


def _dtype_code(x) -> int:
    torch = _torch()
    return _lib.FA_DTYPE_BF16 if x.dtype == torch.bfloat16 else _lib.FA_DTYPE_F32


def covariance_dev(x, mean_f32):
    """(x - mean)^T (x - mean) / n as a float64 (D, D) device tensor (K9)."""
    torch = _torch()
    lib = _lib.load()
    n, dim = x.shape
    cov = torch.empty((dim, dim), dtype=torch.float64, device="cuda")
    check(lib.fa_pca_cov_dev(x.data_ptr(), _dtype_code(x), n, dim, mean_f32.data_ptr(),
                             cov.data_ptr(), None))
    return cov


def pca_train(sample, alpha: float | None = 0.9, d: int | None = None) -> PCAModel:
    """Fit the rotation on the device; keep d components (or the smallest d
    reaching the variance fraction alpha)."""
    data = rows_of(sample)
    n = data.shape[0]
    if n < 2:
        raise ConfigError("need at least 2 vectors to fit a covariance")
    torch = _torch()
    x = as_device_rows(data)
    mean = x.double().mean(0)
    cov = covariance_dev(x, mean.float().contiguous())
    w, v = torch.linalg.eigh(cov)
    eig = torch.clamp(torch.flip(w, [0]), min=0.0)
    basis = torch.flip(v, [1]).contiguous()
    eig_h = eig.cpu().numpy()
    dim = data.shape[1]
    if d is None:
        if alpha is None or not 0.0 < alpha <= 1.0:
            raise ConfigError("variance fraction must lie in (0, 1]")
        total = eig_h.sum()
        if total <= 0:
            d = 1
        else:
            frac = np.cumsum(eig_h) / total
            d = min(int(np.searchsorted(frac, alpha - 1e-12) + 1), dim)
    if not 1 <= d <= dim:
        raise ConfigError(f"retained dimension {d} out of range")
    return PCAModel(mean=mean.cpu().numpy(), basis=basis.cpu().numpy(), eigvals=eig_h, d=int(d))


def _model_dev(model: PCAModel) -> dict:
    """Device copies of the rotation (cached on the model)."""
    cache = getattr(model, "_pca_dev", None)
    if cache is None:
        torch = _torch()
        cache = {
            "mean_f32": torch.from_numpy(model.mean.astype(np.float32)).cuda(),
            "basis_f32": torch.from_numpy(np.ascontiguousarray(model.basis, np.float32)).cuda(),
            "mean_f64": torch.from_numpy(np.ascontiguousarray(model.mean, np.float64)).cuda(),
            "basis_f64": torch.from_numpy(np.ascontiguousarray(model.basis, np.float64)).cuda(),
        }
        model._pca_dev = cache
    return cache


def pca_project_all_dev(model: PCAModel, x, d: int | None = None):
    """(x - mean) @ basis[:, :d] in float32 on the device (K9); x on device or
    host, float32 or a bfloat16 tensor."""
    torch = _torch()
    lib = _lib.load()
    d = model.d if d is None else d
    xd = as_device_rows(x)
    n, dim = xd.shape
    if dim != model.mean.shape[0]:
        raise ConfigError("vector dimension mismatch")
    m = _model_dev(model)
    out = torch.empty((n, d), dtype=torch.float32, device="cuda")
    if n:
        check(lib.fa_pca_project_dev(xd.data_ptr(), _dtype_code(xd), n, dim,
                                     m["mean_f32"].data_ptr(), m["basis_f32"].data_ptr(),
                                     m["basis_f32"].shape[1], d, out.data_ptr(), d, None))
    return out


def pca_project_all(model: PCAModel, data, d: int | None = None) -> np.ndarray:
    return pca_project_all_dev(model, data, d).cpu().numpy()


def pca_project(model: PCAModel, vec, d: int | None = None) -> np.ndarray:
    """Centred projection of one vector (or rows) in float64, like the
    reference (pca.py:57-65)."""
    torch = _torch()
    lib = _lib.load()
    d = model.d if d is None else d
    if d > model.basis.shape[1]:
        raise ConfigError(f"d={d} exceeds basis width")
    v = np.asarray(vec, dtype=np.float64)
    if v.shape[-1] != model.mean.shape[0]:
        raise ConfigError("vector dimension mismatch")
    rows = np.ascontiguousarray(np.atleast_2d(v))
    m = _model_dev(model)
    xd = torch.from_numpy(rows).cuda()
    out = torch.empty((rows.shape[0], d), dtype=torch.float64, device="cuda")
    check(lib.fa_pca_project_f64_dev(xd.data_ptr(), rows.shape[0], rows.shape[1],
                                     m["mean_f64"].data_ptr(), m["basis_f64"].data_ptr(),
                                     m["basis_f64"].shape[1], d, out.data_ptr(), None))
    res = out.cpu().numpy()
    return res if v.ndim > 1 else res[0]
