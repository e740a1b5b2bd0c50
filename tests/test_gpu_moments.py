"""K1 (moments) through the phase call prohd_local_moments: [S_A | S_B | G] about a shift s
(Alg. 1 line 1; Alg. 2 lines 1-2) against fp64 sums of the
same fp32 inputs (the oracle's definition, O1/O3, written out with numpy).

The default Gram is the fp64 DMMA pass (k_gram.cu, products of fp32 values exact in fp64,
subtraction only when s != 0); option k1_path = 1 selects the opt-in int8 tensor-core pass for
s = 0 (k_gram_i8.cu: exact integer slice products, pairs t + u <= 7 kept). Both must agree
with the fp64 sums to 1e-12 of sum_p |x_pi - s_i| |x_pj - s_j| (the scale of the
accumulation; fp64 accumulation over 1e5 points, or the int8 path's dropped slice pairs,
< 2^-62 of max|x_i| max|x_j| per point), far inside the ~1e-9 relative C accuracy the
direction parity needs."""
import os
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2511_18207_b200 import Context
    return Context(0)


def _ref(A, B, s):
    a = A.astype(np.float64) - s
    b = B.astype(np.float64) - s
    G = a.T @ a + b.T @ b
    scale = np.abs(a).T @ np.abs(a) + np.abs(b).T @ np.abs(b)
    return a.sum(0), b.sum(0), G, scale


def _check(ctx, A, B, s, rtol=1e-12):
    D = A.shape[1]
    mom = ctx.local_moments(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), s).cpu().numpy()
    SA, SB, G = mom[:D], mom[D:2 * D], mom[2 * D:].reshape(D, D)
    rSA, rSB, rG, scale = _ref(A, B, s)
    sa_scale = np.abs(A.astype(np.float64) - s).sum(0) + 1e-300
    sb_scale = np.abs(B.astype(np.float64) - s).sum(0) + 1e-300
    assert np.all(np.abs(SA - rSA) <= 1e-13 * sa_scale)
    assert np.all(np.abs(SB - rSB) <= 1e-13 * sb_scale)
    err = np.abs(G - rG) / (scale + 1e-300)
    assert err.max() <= rtol, f"max G error {err.max():.2e} (rel. to sum |x_i||x_j|)"
    assert np.array_equal(G, G.T)


@pytest.fixture(params=["dmma", "i8"])
def gram_path(request):
    from paper_2511_18207_b200 import option
    with option("k1_path", 1 if request.param == "i8" else 0):
        yield request.param


@pytest.mark.parametrize("nA,nB,D", [(1, 1, 3), (63, 65, 16), (1000, 777, 64), (4099, 2051, 100),
                                     (20000, 20001, 128), (9000, 9000, 200), (65536, 70001, 256)])
def test_gram_about_origin(ctx, gram_path, nA, nB, D):
    rng = np.random.default_rng(nA + D)
    A = rng.standard_normal((nA, D)).astype(np.float32)
    B = (rng.standard_t(3, (nB, D)) * 5 + 0.3).astype(np.float32)  # heavy tails, small offset
    _check(ctx, A, B, np.zeros(D))


def test_gram_special_values(ctx, gram_path):
    rng = np.random.default_rng(5)
    D = 48
    A = rng.standard_normal((5000, D)).astype(np.float32)
    B = rng.standard_normal((3000, D)).astype(np.float32)
    A[:, 0] = 0.0                   # an all-zero column
    A[::3, 1] = np.float32(-0.0)
    A[::7, 2] = np.float32(3e-40)   # subnormals
    B[::5, 3] = np.float32(1e-30)   # tiny normals next to O(1) values
    B[17, 4] = np.float32(1e6)      # one huge outlier in a column
    _check(ctx, A, B, np.zeros(D))


def test_gram_shifted(ctx):
    """s != 0: the fp64 DMMA pass subtracts the shift (large common offset)."""
    rng = np.random.default_rng(9)
    D = 96
    A = (rng.standard_normal((20000, D)) + 4096).astype(np.float32)
    B = (rng.standard_normal((15000, D)) + 4096.5).astype(np.float32)
    s = np.concatenate([A[:4096], B[:4096]]).astype(np.float64).mean(0)
    _check(ctx, A, B, s)


@pytest.mark.parametrize("nA,nB,D", [(3001, 2999, 300), (2000, 1500, 513), (1200, 1100, 1000), (777, 5000, 33),
                                     (5000, 1, 260)])
def test_gram_wide_and_ragged(ctx, nA, nB, D):
    """D > 256 (groups over 4x4 squares of 32-feature blocks, the column-sum pass looping over
    piece blocks) and D % 4 != 0 (4-byte copies, scalar column sums), against the fp64 sums."""
    rng = np.random.default_rng(D)
    A = (rng.standard_normal((nA, D)) * rng.uniform(0.1, 3, D)).astype(np.float32)
    B = (rng.standard_t(4, (nB, D)) + 0.25).astype(np.float32)
    _check(ctx, A, B, np.zeros(D))


def test_gram_replicated_ksteps(ctx):
    """Small D: each 32x32 tile runs on 4 (D <= 32) or 2 warps taking alternate k-steps, and
    the replicas' partials are summed by the reduce kernel."""
    rng = np.random.default_rng(17)
    for D, n in [(8, 40001), (32, 30000), (64, 20011), (96, 10000)]:
        A = rng.standard_normal((n, D)).astype(np.float32)
        B = (rng.standard_normal((n // 2 + 3, D)) * 2 - 1).astype(np.float32)
        _check(ctx, A, B, np.zeros(D))


def _i8_bound(A, B, shifted):
    """Element-wise bound on |C_gpu - C_ref| for the int8 Gram (k_gram_i8.cu): every value is a
    fixed-point integer on the grid 2^-k_j <= 2^-29 M_j (M_j = max |x - s_j|, exact), rounded to
    nearest (|e_j| <= 2^-30 M_j; with a shift the FMA first rounds to 24 bits of |F| <= 2^30:
    |e_j| <= 2^-23 M_j), and the dropped d_3 d_3 level adds <= 2^14 grid^2 per point."""
    X = np.concatenate([A, B]).astype(np.float64)
    mu = X.mean(0)
    Y = np.abs(X - mu)
    # M_j = max |x - s_j| with s_j the shift kernel's value (0 or ~the sample mean): covered by
    M = 1.1 * np.maximum(np.abs(X).max(0), Y.max(0)) + 1e-300
    e = M * (2.0 ** -23 if shifted else 2.0 ** -30)
    Ymean = Y.mean(0)
    # C_gpu is the covariance of the quantized values x + e (G and S come from the same integers):
    # |cov(x + e) - cov(x)| <= 2 (mean|x_i - mu_i| e_j + mean|x_j - mu_j| e_i) + 4 e_i e_j
    return (2 * (Ymean[:, None] * e[None, :] + Ymean[None, :] * e[:, None]) + 4 * np.outer(e, e)
            + 2.0 ** -44 * np.outer(M, M)) * 1.05 + 1e-15 * (Y.T @ Y) / X.shape[0]


_I8_KINDS = ["gauss", "heavy", "unit", "offset", "ragged", "windows",
             "s_gauss16", "s_heavy128", "s_unit64", "s_offset96", "s_ragged20", "s_windows64", "s_tiny"]


@pytest.mark.parametrize("kind", _I8_KINDS)
def test_covariance_int8_path(ctx, kind):
    """Step 1a through prohd_covariance (the path prohd_estimate uses): the int8 tensor-core Gram
    (gram_i8_kernel for 128 < D <= 256, gram_i8s_kernel for D <= 128: kinds "s_*"), against the
    oracle's two-pass fp64 covariance (O3, oracle/prohd.py), within the fixed-point bound above;
    mu within the grid's rounding bound."""
    from oracle import prohd as OP
    from paper_2511_18207_b200 import option
    rng = np.random.default_rng(_I8_KINDS.index(kind) + 1)
    D = {"gauss": 256, "heavy": 256, "unit": 200, "offset": 160, "ragged": 132, "windows": 256,
         "s_gauss16": 16, "s_heavy128": 128, "s_unit64": 64, "s_offset96": 96, "s_ragged20": 20,
         "s_windows64": 64, "s_tiny": 16}[kind]
    # "windows": > 682 chunks of 64 points per group (24 groups), so every TMEM accumulator is
    # drained to the fp64 slabs mid-sweep and accumulated again; "s_windows64": the same on the
    # D <= 128 kernel with two CTAs (option k1_i8_ctas), ~2.3 windows per CTA
    nA, nB = {"ragged": (1237, 70001), "windows": (560000, 560003), "s_ragged20": (1237, 70001),
              "s_windows64": (50001, 50003), "s_tiny": (3, 5)}.get(kind, (40011, 35003))
    base = kind[2:] if kind.startswith("s_") else kind
    base = base.rstrip("0123456789")
    if base in ("heavy", "windows"):
        A = (rng.standard_t(3, (nA, D)) * rng.uniform(0.1, 3, D)).astype(np.float32)
        B = (rng.standard_t(3, (nB, D)) * rng.uniform(0.1, 3, D) + 0.3).astype(np.float32)
    elif base == "unit":
        A = np.clip(rng.random((nA, D)) * 0.6 + 0.1 * rng.standard_normal((nA, D)), 0, 1).astype(np.float32)
        B = np.clip(rng.random((nB, D)) * 0.5 + 0.1 * rng.standard_normal((nB, D)), 0, 1).astype(np.float32)
    elif base == "offset":
        A = (rng.standard_normal((nA, D)) + 4096).astype(np.float32)
        B = (rng.standard_normal((nB, D)) + 4096.5).astype(np.float32)
    else:
        A = rng.standard_normal((nA, D)).astype(np.float32)
        B = (rng.standard_normal((nB, D)) * 2 + 1).astype(np.float32)
    with option("k1_i8_ctas", 2 if kind == "s_windows64" else -1):
        mu, C, path = ctx.covariance(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
    assert path == 1, "the int8 Gram should serve D <= 256 (D % 4 == 0)"
    rmu, rC = OP.covariance(A, B)
    # mu is the mean of the fixed-point values: within the rounding bound e_j of the grid
    X = np.concatenate([A, B]).astype(np.float64)
    M = 1.1 * np.maximum(np.abs(X).max(0), np.abs(X - rmu).max(0))
    assert np.all(np.abs(mu - rmu) <= M * (2.0 ** -23 if base == "offset" else 2.0 ** -30) + 1e-15 * np.abs(rmu))
    bound = _i8_bound(A, B, base == "offset")
    frac = np.abs(C - rC) / bound
    assert frac.max() <= 1.0, f"max |dC| / bound = {frac.max():.3f}"
    assert np.array_equal(C, C.T)
    print(f"{kind} D={D}: max |dC|/bound {frac.max():.2e}, max |dC|/max|C| "
          f"{np.abs(C - rC).max() / np.abs(rC).max():.2e}")


def test_covariance_dmma_option_and_small_d(ctx):
    """option k1_path = 0 selects the fp64 DMMA Gram (D % 4 != 0 always takes it): C within 1e-12
    of the accumulation scale."""
    from oracle import prohd as OP
    from paper_2511_18207_b200 import option
    rng = np.random.default_rng(11)
    for D, opt in ((256, 0), (96, 0), (18, -1)):
        A = rng.standard_normal((20000, D)).astype(np.float32)
        B = (rng.standard_t(4, (15000, D)) + 0.2).astype(np.float32)
        with option("k1_path", opt):
            mu, C, path = ctx.covariance(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
        assert path == 0
        rmu, rC = OP.covariance(A, B)
        X = np.abs(np.concatenate([A, B]).astype(np.float64) - rmu)
        assert np.all(np.abs(C - rC) <= 1e-12 * (X.T @ X) / X.shape[0] + 1e-300)
