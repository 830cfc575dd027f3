"""Rotation used by the Flash coder (flashann/providers/pca.py:27-71), on the GPU.

pca_train: float64 mean, float32 centred covariance GEMM (cuBLAS, TF32 off,
like the reference's fp32 sgemm), float64 symmetric eigendecomposition
(cuSOLVER), components by descending eigenvalue, eigenvalues clamped at 0.
pca_project_all: float32 (x - mean) @ basis[:, :d] on the device.

Eigenvectors are defined up to sign (and up to rotation inside degenerate
eigenspaces); everything downstream (codes, tables, the graph) is invariant
to a per-component sign, and parity tests compare bases up to sign.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._arrays import is_tensor, rows_of
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
    torch.backends.cuda.matmul.allow_tf32 = False
    return torch


def as_device_f32(data):
    torch = _torch()
    if is_tensor(data):
        return data.to(device="cuda", dtype=torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(data, dtype=np.float32)).cuda()


def pca_train(sample, alpha: float | None = 0.9, d: int | None = None) -> PCAModel:
    """Fit the rotation on the device; keep d components (or the smallest d
    reaching the variance fraction alpha)."""
    data = rows_of(sample)
    n = data.shape[0]
    if n < 2:
        raise ConfigError("need at least 2 vectors to fit a covariance")
    torch = _torch()
    x = as_device_f32(data)
    mean = x.double().mean(0)
    xc = x - mean.float()
    cov = (xc.T @ xc).double() / n
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


def pca_project_all_dev(model: PCAModel, x, d: int | None = None):
    """(x - mean) @ basis[:, :d] in float32 on the device; x on device or host."""
    torch = _torch()
    d = model.d if d is None else d
    xd = as_device_f32(x)
    mean = torch.from_numpy(model.mean.astype(np.float32)).cuda()
    b = torch.from_numpy(np.ascontiguousarray(model.basis[:, :d], dtype=np.float32)).cuda()
    return ((xd - mean) @ b).contiguous()


def pca_project_all(model: PCAModel, data, d: int | None = None) -> np.ndarray:
    return pca_project_all_dev(model, data, d).cpu().numpy()


def pca_project(model: PCAModel, vec, d: int | None = None) -> np.ndarray:
    """Centred projection of one vector (float64, like the reference)."""
    torch = _torch()
    d = model.d if d is None else d
    if d > model.basis.shape[1]:
        raise ConfigError(f"d={d} exceeds basis width")
    v = np.asarray(vec, dtype=np.float64)
    if v.shape[-1] != model.mean.shape[0]:
        raise ConfigError("vector dimension mismatch")
    vd = torch.from_numpy(v).cuda()
    out = (vd - torch.from_numpy(model.mean).cuda()) @ torch.from_numpy(model.basis[:, :d]).cuda()
    return out.cpu().numpy()
