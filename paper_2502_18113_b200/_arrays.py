"""Array plumbing shared by the host modules."""

from __future__ import annotations

import numpy as np


def is_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def rows_of(x):
    """The (n, dim) matrix behind a VectorDataset, ndarray or torch tensor."""
    if isinstance(x, np.ndarray) or is_tensor(x):
        return x
    return x.data
