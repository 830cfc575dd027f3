"""GPU: the standalone block scan (K1, direct loads and TMA-staged) against the
oracle's fa_batch_lanes restatement on the padded device block layout."""

import numpy as np
import pytest

from oracle import native

pytestmark = pytest.mark.gpu


def _layout(cap, m):
    nb = (cap + 15) // 16
    codes_off = (16 + 4 * cap + 15) // 16 * 16
    stride = (codes_off + nb * m * 16 + 127) // 128 * 128
    return nb, codes_off, stride


def _expected(adt, blocks, sel, cap, m, codes_off):
    nb = (cap + 15) // 16
    out = np.empty(sel.shape[0], np.uint64)
    for q in range(sel.shape[0]):
        best = np.uint64(~np.uint64(0))
        for b in sel[q]:
            blk = blocks[b]
            cnt = min(int(blk[:4].view(np.int32)[0]), cap)
            ids = blk[16: 16 + 4 * cap].view(np.int32)
            lanes = native.batch_lanes(adt[q], blk[codes_off: codes_off + nb * m * 16], nb)
            for j in range(cnt):
                if ids[j] >= 0:
                    k = np.uint64((int(lanes[j]) << 32) | int(ids[j]))
                    best = min(best, k)
        out[q] = best
    return out


@pytest.mark.parametrize("cap,m", [(32, 32), (64, 64), (64, 48), (96, 96), (16, 8), (64, 80), (32, 112)])
def test_scan_select_matches_oracle(cuda, cap, m):
    import ctypes

    from paper_2502_18113_b200 import _lib

    torch = cuda
    lib = _lib.load()
    nb, codes_off, stride = _layout(cap, m)
    rng = np.random.default_rng(cap + m)
    nblocks, nq, ns = 3000, 37, 45
    blocks = rng.integers(0, 16, size=(nblocks, stride), dtype=np.uint8)
    counts = rng.integers(0, cap + 1, nblocks).astype(np.int32)
    blocks[:, :4] = counts.view(np.uint8).reshape(-1, 4)
    ids = rng.integers(-1, 1 << 20, size=(nblocks, cap)).astype(np.int32)
    blocks[:, 16: 16 + 4 * cap] = ids.view(np.uint8).reshape(nblocks, -1)
    adt = rng.integers(0, 256 // max(1, m // 8), size=(nq, m, 16), dtype=np.uint8)
    sel = rng.integers(0, nblocks, size=(nq, ns)).astype(np.int32)
    expect = _expected(adt, blocks, sel, cap, m, codes_off)
    db, da, ds = (torch.from_numpy(x).cuda() for x in (blocks, adt, sel))
    for fn in (lib.fa_scan_select_dev, lib.fa_scan_select_tma_dev):
        out = torch.empty(nq, dtype=torch.int64, device="cuda")
        _lib.check(fn(da.data_ptr(), nq, db.data_ptr(), nblocks, stride, codes_off, cap, m,
                      ds.data_ptr(), ns, out.data_ptr(), None))
        got = out.cpu().numpy().view(np.uint64)
        assert np.array_equal(got, expect), fn.__name__
    del ctypes
