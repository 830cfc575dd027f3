"""Boundary helpers for the reference's interleaved vertex blocks.

The reference keeps one row per (vertex, layer) (flashann/layout.py:1-45):
``[int32 count | int32 ids x cap (-1 empty) | u8 codes: ceil(cap/16) batches
x m subspaces x 16 lanes]``.  The device graph is structure-of-arrays instead
(id rows + counts + one flat code table, csrc/search.cuh); these vectorised
helpers only describe/convert the reference rows exchanged at the boundary.
"""

from __future__ import annotations

import numpy as np

LANES = 16


def batches_for(cap: int) -> int:
    return (cap + LANES - 1) // LANES


def block_stride(cap: int, m: int) -> int:
    """Reference row width in bytes (flashann/layout.py:30-32)."""
    return 4 * (1 + cap) + batches_for(cap) * m * LANES


def codes_offset(cap: int) -> int:
    return 4 * (1 + cap)


def empty_rows(rows: int, cap: int, m: int) -> np.ndarray:
    """Rows with count 0, every id slot -1 and zero codes."""
    out = np.zeros((rows, block_stride(cap, m)), dtype=np.uint8)
    out[:, 4 : codes_offset(cap)] = 0xFF  # int32 -1 in every id slot
    return out


def row_ids(blocks: np.ndarray, row: int, cap: int) -> np.ndarray:
    cnt = int(blocks[row, :4].view(np.int32)[0])
    return blocks[row, 4 : codes_offset(cap)].view(np.int32)[: max(0, min(cnt, cap))].copy()


def set_row(blocks: np.ndarray, row: int, cap: int, m: int, ids, codes=None) -> None:
    """Write one row: ids (len <= cap) and, when m > 0, the codes (len, m)."""
    ids = np.asarray(ids, dtype=np.int32).reshape(-1)
    if ids.size > cap:
        raise ValueError(f"{ids.size} neighbours exceed capacity {cap}")
    slots = np.full(cap, -1, dtype=np.int32)
    slots[: ids.size] = ids
    blocks[row, 4 : codes_offset(cap)] = slots.view(np.uint8)
    if m:
        if codes is None:
            raise ValueError("a coded row needs the neighbours' codes")
        lanes = np.zeros((batches_for(cap) * LANES, m), dtype=np.uint8)
        lanes[: ids.size] = np.asarray(codes, dtype=np.uint8).reshape(ids.size, m)
        # (batch, lane, sub) -> (batch, sub, lane): subspace-major 16-lane groups
        grp = lanes.reshape(batches_for(cap), LANES, m).transpose(0, 2, 1)
        blocks[row, codes_offset(cap):] = grp.reshape(-1)
    blocks[row, :4] = np.array([ids.size], dtype=np.int32).view(np.uint8)


def row_codes(blocks: np.ndarray, row: int, cap: int, m: int) -> np.ndarray:
    """Codes of the live slots, (count, m) in slot order."""
    cnt = int(blocks[row, :4].view(np.int32)[0])
    grp = blocks[row, codes_offset(cap):].reshape(batches_for(cap), m, LANES)
    return grp.transpose(0, 2, 1).reshape(-1, m)[:cnt].copy()
