"""K9: the PCA contractions on the tensor cores (csrc/pca_gemm.cu) against the
reference's numpy arithmetic (flashann/providers/pca.py:27-71).

* covariance and projection GEMMs (3xTF32 tcgen05) against float64 numpy of
  the same float32-centred operands: relative error <= 2e-6, f32 and bf16
  rows, widths that exercise the zero-padded TMA paths (D not a multiple of
  4, D < 128, n not a multiple of the 128-row tile);
* config 4's 960 -> 256 PCA against the reference's own pca_train output
  (tests/golden/gen_pca_golden.py): mean 1e-12, eigenvalues 1e-6 of the
  largest, every one of the 256 basis columns up to sign with
  1 - |cos| <= 1e-6, and pca_project_all of 64 rows within 1e-5 of the
  reference's own fp32 sgemm (sign-aligned);
* pca_project (float64 single vectors) against numpy float64;
* the covariance's K splits at the real sample sizes (each owns a k-block;
  bitwise stable after other tensor-core work left TMEM dirty).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _centred(x, mean32):
    return (x.astype(np.float32) - mean32).astype(np.float32)


@pytest.mark.parametrize("n,D", [(1000, 128), (777, 24), (3000, 960), (257, 130), (64, 7)])
@pytest.mark.parametrize("bf16", [False, True])
def test_covariance_gemm(cuda, n, D, bf16):
    torch = cuda
    from paper_2502_18113_b200 import pca

    rng = np.random.default_rng(n + D)
    x = (rng.normal(size=(n, D)) * rng.uniform(0.1, 3.0, D) + rng.normal(size=D)).astype(np.float32)
    xt = torch.from_numpy(x).cuda()
    if bf16:
        xt = xt.to(torch.bfloat16)
        x = xt.float().cpu().numpy()
    mean32 = x.astype(np.float64).mean(0).astype(np.float32)
    cov = pca.covariance_dev(xt, torch.from_numpy(mean32).cuda()).cpu().numpy()
    xc = _centred(x, mean32).astype(np.float64)
    ref = xc.T @ xc / n
    scale = np.sqrt(np.outer(np.diag(ref), np.diag(ref))) + 1e-30
    assert np.abs(cov - ref).max() / np.abs(ref).max() <= 2e-6
    assert (np.abs(cov - ref) / scale).max() <= 1e-5
    assert np.array_equal(cov, cov.T)


@pytest.mark.parametrize("n", [20000, 100000])
def test_covariance_after_other_tmem_work(cuda, n):
    """Sample sizes whose k-block count does not divide evenly over the
    K splits (20,000 rows = config 1's whole sample, 100,000 = the training
    sample of configs 2-5, D = 128: one output tile, up to 2 x 148 splits).
    Every split must own a k-block: an empty one would drain whatever an
    earlier kernel left in TMEM into the sum.  A projection with large values
    runs first, so such leftovers would be large; the covariance must match
    float64 numpy and be bitwise stable across calls."""
    torch = cuda
    from paper_2502_18113_b200 import pca

    rng = np.random.default_rng(n)
    # enough row tiles for a persistent CTA on every SM
    g = torch.Generator(device="cuda").manual_seed(n)
    big = torch.randn((300_000, 128), generator=g, device="cuda") * 1e4
    q, _ = np.linalg.qr(rng.normal(size=(128, 128)))
    junk = pca.PCAModel(mean=np.zeros(128), basis=q, eigvals=np.ones(128), d=128)
    x = rng.normal(size=(n, 128)).astype(np.float32)
    xt = torch.from_numpy(x).cuda()
    mean32 = x.astype(np.float64).mean(0).astype(np.float32)
    mt = torch.from_numpy(mean32).cuda()
    covs = []
    for _ in range(3):
        pca.pca_project_all_dev(junk, big)  # leaves large accumulators in TMEM
        covs.append(pca.covariance_dev(xt, mt).cpu().numpy())
    xc = _centred(x, mean32).astype(np.float64)
    ref = xc.T @ xc / n
    assert np.abs(covs[0] - ref).max() / np.abs(ref).max() <= 2e-6
    assert all(np.array_equal(c, covs[0]) for c in covs[1:])


@pytest.mark.parametrize("n,D,d", [(1000, 128, 128), (1500, 960, 256), (700, 768, 300),
                                   (129, 24, 16), (50, 96, 96), (333, 130, 129)])
@pytest.mark.parametrize("bf16", [False, True])
def test_projection_gemm(cuda, n, D, d, bf16):
    torch = cuda
    from paper_2502_18113_b200 import pca

    rng = np.random.default_rng(n * 7 + D + d)
    x = rng.normal(size=(n, D)).astype(np.float32) * 3 + 1
    xt = torch.from_numpy(x).cuda()
    if bf16:
        xt = xt.to(torch.bfloat16)
        x = xt.float().cpu().numpy()
    q, _ = np.linalg.qr(rng.normal(size=(D, D)))
    model = pca.PCAModel(mean=rng.normal(size=D), basis=q, eigvals=np.ones(D), d=d)
    out = pca.pca_project_all_dev(model, xt).cpu().numpy()
    mean32 = model.mean.astype(np.float32)
    ref = _centred(x, mean32).astype(np.float64) @ q[:, :d].astype(np.float32).astype(np.float64)
    rown = np.linalg.norm(_centred(x, mean32).astype(np.float64), axis=1)[:, None]
    assert out.shape == (n, d)
    assert (np.abs(out - ref) / rown).max() <= 2e-6


def test_config4_pca_matches_reference(cuda):
    from pathlib import Path

    from paper_2502_18113_b200 import dataset, pca

    g = np.load(Path(__file__).parent / "golden" / "pca_c4_golden.npz")
    x, _ = dataset.baseline_config(4, n=6000, nq=0)
    model = pca.pca_train(x, d=256)
    assert np.allclose(model.mean, g["mean"], rtol=0, atol=1e-12)
    lam0 = g["eigvals"][0]
    # 1e-6 of the largest: the tensor core's truncating fp32 accumulator
    # leaves a ~1e-7 relative low bias (the reference's own fp32 sgemm has
    # ~3e-7 elementwise error)
    assert np.abs(model.eigvals - g["eigvals"]).max() <= 1e-6 * lam0
    b = model.basis[:, :256]
    cos = (b * g["basis"].astype(np.float64)).sum(0)
    assert (1.0 - np.abs(cos)).max() <= 1e-6
    # the reference's pca_project_all (its own sgemm) of 64 rows, sign-aligned
    proj = pca.pca_project_all(model, x[:64])
    proj *= np.sign(cos)[None, :].astype(np.float32)
    scale = np.linalg.norm(x[:64] - model.mean.astype(np.float32), axis=1)[:, None]
    # (includes the basis difference of the small-gap columns; the GEMM itself
    # is held to 2e-6 against float64 in test_projection_gemm)
    assert (np.abs(proj - g["proj64"]) / scale).max() <= 1e-5


def test_single_vector_projection_f64(cuda):
    from paper_2502_18113_b200 import pca

    rng = np.random.default_rng(5)
    D = 40
    q, _ = np.linalg.qr(rng.normal(size=(D, D)))
    model = pca.PCAModel(mean=rng.normal(size=D), basis=q, eigvals=np.ones(D), d=12)
    v = rng.normal(size=D)
    out = pca.pca_project(model, v)
    ref = (v - model.mean) @ q[:, :12]
    assert out.shape == (12,)
    assert np.allclose(out, ref, rtol=0, atol=1e-13)
    rows = rng.normal(size=(5, D))
    assert np.allclose(pca.pca_project(model, rows, d=D), (rows - model.mean) @ q, atol=1e-13)
