"""Exact strategy provider (kind 0): fp32 L2 over the raw vectors.

Mirrors the reference's ExactProvider (flashann/providers/exact.py): no
training, no codes (code_subspaces = 0), core arrays {"vecs", "dim"}, the
query payload is the query vector itself.  The distances come from the
device index's exact kind (a device index created with m = 0).
"""

from __future__ import annotations

import numpy as np

from ._arrays import is_tensor, rows_of
from .pca import as_device_f32


class ExactProvider:
    kind = "exact"
    kind_id = 0
    code_subspaces = 0

    def __init__(self):
        self.dataset = None
        self.dev: dict = {}

    def attach(self, dataset, vecs_dev=None) -> None:
        self.dataset = dataset
        data = rows_of(dataset)
        self.dev = {"vecs": vecs_dev if vecs_dev is not None else as_device_f32(data)}

    def core_arrays(self) -> dict:
        data = rows_of(self.dataset)
        if is_tensor(data):
            data = data.cpu().numpy()
        data = np.ascontiguousarray(data, dtype=np.float32)
        return {"vecs": data, "dim": data.shape[1]}

    def query_aux(self, queries) -> np.ndarray:
        return np.ascontiguousarray(np.atleast_2d(queries), dtype=np.float32)

    def query_aux_dev(self, queries_dev):
        return queries_dev

    def state_dict(self) -> dict:
        return {}

    @classmethod
    def from_state(cls, state: dict) -> "ExactProvider":
        return cls()
