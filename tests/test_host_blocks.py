"""Reference blocks written on the host cores (fa_assemble_blocks: the host
drop-in's output path) against the layout helpers' own row writer
(layout.set_row, flashann/layout.py:63-94), byte for byte.  No device needed."""

import ctypes as C

import numpy as np
import pytest

from paper_2502_18113_b200 import _lib, layout


@pytest.mark.parametrize("cap,m", [(16, 32), (32, 64), (64, 64), (64, 48), (96, 96), (20, 20),
                                   (33, 7)])
def test_assemble_matches_layout(cap, m):
    rng = np.random.default_rng(cap * 131 + m)
    n, rows = 500, 257
    codes = rng.integers(0, 16, size=(n, m), dtype=np.uint8)
    packed = np.full((rows, 1 + cap), -1, dtype=np.int32)
    ref = layout.empty_rows(rows, cap, m)
    for r in range(rows):
        cnt = int(rng.integers(0, cap + 1)) if r % 7 else cap
        ids = rng.choice(n, size=cnt, replace=False).astype(np.int32)
        packed[r, 0] = cnt
        packed[r, 1:1 + cnt] = ids
        layout.set_row(ref, r, cap, m, ids, codes[ids])
    out = np.full_like(ref, 0xAB)
    lib = _lib.load(require_device=False)
    _lib.check(lib.fa_assemble_blocks(out.ctypes.data, rows, out.shape[1], cap, m,
                                      packed.ctypes.data, codes.ctypes.data, n))
    np.testing.assert_array_equal(out, ref)


def test_assemble_rejects_short_stride():
    lib = _lib.load(require_device=False)
    buf = np.zeros((1, 8), np.uint8)
    packed = np.zeros((1, 17), np.int32)
    codes = np.zeros((1, 32), np.uint8)
    with pytest.raises(ValueError):
        _lib.check(lib.fa_assemble_blocks(buf.ctypes.data, 1, 8, 16, 32, packed.ctypes.data,
                                          codes.ctypes.data, 1))
