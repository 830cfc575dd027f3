"""GPU parity of the table kernels against the oracle and the reference's
golden outputs (bit-exact: integer/byte work, and the pinned fp32 tree)."""

import hashlib

import numpy as np
import pytest

import golden_inputs as gi
from oracle import native

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def core(cuda):
    from paper_2502_18113_b200 import sm100

    return sm100


@pytest.mark.parametrize("m", gi.SCAN_MS)
def test_scan_cases_bit_exact(core, golden, m):
    adts, codes = gi.scan_cases(m)
    got = core.flash_batch_distance_many(adts, codes)
    assert np.array_equal(got[:256], golden[f"scan_{m}_head"])
    assert sha(got) == str(golden[f"scan_{m}_sha"])


def test_scan_saturation_extremes(core):
    m = 96
    adts = np.full((4, m, 16), 255, np.uint8)
    adts[1] = 0
    adts[2] = 2  # 96*2 = 192 < 255: no saturation
    adts[3, :, 0] = 3  # 288 on lane-code 0 -> 255
    codes = np.zeros((4, m, 16), np.uint8)
    out = core.flash_batch_distance_many(adts, codes)
    assert (out[0] == 255).all() and (out[1] == 0).all() and (out[2] == 192).all()
    assert (out[3] == 255).all()


def test_scan_blocks(core, golden):
    adt, flat = gi.block_case()
    assert np.array_equal(core.flash_batch_blocks(adt, flat, 4), golden["blocks"])
    one = core.flash_batch_distance(adt, flat[: 16 * 16].reshape(16, 16))
    assert np.array_equal(one, golden["blocks"][:16])


def test_quantizer(core, golden):
    d, dmin, delta = gi.quantize_inputs()
    assert np.array_equal(core.quantize_distance(d, dmin, delta), golden["quant"])
    assert core.quantize_distance(dmin + delta / 2, dmin, delta) == 127


@pytest.mark.parametrize("d", gi.L2_DIMS)
def test_l2_tree(core, golden, d):
    a, b = gi.l2_inputs(d)
    got = np.array([core.l2sq_f32(x, y) for x, y in zip(a[:8], b[:8])])
    assert np.array_equal(got, golden[f"l2_{d}"][:8])


@pytest.mark.parametrize("name", list(gi.MODELS))
def test_encoder_bit_exact(core, golden, name):
    p = f"model_{name}_"
    cent, dims, offs = golden[p + "cent"], golden[p + "dims"], golden[p + "offs"]
    dmin, dmax = golden[p + "range"]
    red = gi.encode_inputs(cent, dims, gi.MODELS[name])
    codes, adts = core.flash_encode_adt_many(cent, dims, offs, dmin, dmax - dmin, red)
    assert np.array_equal(codes, golden[p + "enc_codes"])
    assert np.array_equal(adts, golden[p + "enc_adt"])
    red_u, dmins, deltas = gi.ulp_inputs(cent, dims, offs, gi.MODELS[name])
    for r in range(0, red_u.shape[0], 7):
        c, a = core.flash_encode_adt(cent, dims, offs, dmins[r], deltas[r], red_u[r])
        assert np.array_equal(c, golden[p + "ulp_codes"][r])
        assert np.array_equal(a, golden[p + "ulp_adt"][r])


def test_sdt_sums_and_select(core, golden):
    sdt = golden["model_c1s_sdt"]
    codes = gi.select_codes(sdt.shape[0])
    a, b = gi.sdt_pairs(codes)
    got = np.array([core.flash_sdt_distance(sdt, x, y) for x, y in zip(a[:64], b[:64])])
    assert np.array_equal(got, golden["sdt_sums"][:64])
    prov = {"codes": codes, "sdt": sdt}
    outs = []
    for ids, d, cap in gi.select_cases(codes, sdt):
        outs.append(np.array(core.select_neighbors(4, prov, ids, d, cap) + [-2], np.int32))
    assert np.array_equal(np.concatenate(outs), golden["select_out"])


def test_select_asymmetric_table_matches_oracle(core):
    """Hook contract holds for arbitrary (non-symmetric) tables too."""
    rng = np.random.default_rng(5)
    m = 24
    sdt = rng.integers(0, 20, size=(m, 16, 16), dtype=np.uint8)
    codes = rng.integers(0, 16, size=(300, m), dtype=np.uint8)
    for t in range(20):
        nc = int(rng.integers(5, 90))
        ids = rng.choice(300, nc, replace=False).astype(np.int32)
        d = np.sort(rng.integers(100, 300, nc)).astype(np.float64)
        cap = int(rng.integers(1, 40))
        assert core.select_neighbors(4, {"codes": codes, "sdt": sdt}, ids, d, cap) == \
            native.select(sdt, codes, ids, d, cap)


@pytest.mark.parametrize("dims_per", [1, 2, 3, 4, 8, 5])
def test_encoder_threshold_quantiser_random_ranges(core, dims_per):
    """K2's quantiser runs as per-coder float thresholds (csrc/encode.cu); the
    tables must equal the oracle's IEEE-double formula (fa_quantize,
    _simd.h:99-107) for arbitrary ranges: 40 random (dist_min, delta) pairs,
    including tiny and huge deltas and dist_min above some distances, over
    rows whose distances spread across the whole range.  Uniform and
    non-uniform subspace widths (5 dims: the generic, non-unrolled path)."""
    rng = np.random.default_rng(dims_per)
    m = 12
    dims = np.full(m, dims_per, np.int32)
    if dims_per == 5:
        dims[::3] = 4  # a split with two widths
    offs = np.concatenate([[0], np.cumsum(dims)[:-1]]).astype(np.int32)
    dmax = int(dims.max())
    cent = np.zeros((m, 16, dmax), np.float32)
    for i in range(m):
        cent[i, :, :dims[i]] = rng.normal(size=(16, dims[i])) * rng.uniform(0.1, 10)
    red = (rng.normal(size=(64, int(dims.sum()))) * rng.uniform(0.1, 10, 64)[:, None]).astype(np.float32)
    for t in range(40):
        scale = 10.0 ** rng.uniform(-3, 3)
        dmin = float(rng.uniform(0, 2) * scale) if t % 4 else 0.0
        delta = float(10.0 ** rng.uniform(-4, 4)) * scale
        c_gpu, a_gpu = core.flash_encode_adt_many(cent, dims, offs, dmin, delta, red)
        c_or, a_or = native.encode_adt(red, cent, dims, offs, dmin, delta)
        assert np.array_equal(np.asarray(c_gpu).reshape(c_or.shape), c_or), (t, dmin, delta)
        assert np.array_equal(np.asarray(a_gpu).reshape(a_or.shape), a_or), (t, dmin, delta)
