"""K3 (projection) through the test hook prohd_project: the fp32 projections the selection
starts from (Alg. 1 line 4 / Alg. 2 line 5; pi = x^T u)
against the exact fp64 dot products of the same fp32 points and fp64 directions (the oracle's
O6 arithmetic written out with numpy).

The selection is exact whatever the projection error, as long as the guard band of K4 holds:
|pi32 - pi64| <= eps for every point and direction. These tests assert that
bound element by element on the BASELINE generators, ragged shapes, both K3 variants (the
tcgen05 3xTF32 kernel for D % 4 == 0, D <= 256, and the SIMT kernels otherwise), and report
how much of the bound the measured error uses."""
import os

import numpy as np
import pytest
import torch

import datagen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2511_18207_b200 import Context
    return Context(0)


def _dirs(D, L, seed):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((D, max(L, 1))))
    return np.ascontiguousarray(Q[:, :L].T)  # L x D, orthonormal rows


def _check(ctx, X, U):
    P, eps = ctx.project(torch.from_numpy(X).cuda(), U)
    P = P.cpu().numpy().astype(np.float64)
    ref = U @ X.astype(np.float64).T  # L x n, exact up to fp64 rounding (~1e-16 ||x||)
    err = np.abs(P - ref)
    assert np.all(np.isfinite(P))
    assert err.max() <= eps, f"max |pi32 - pi64| {err.max():.3e} > eps {eps:.3e}"
    nrm = np.sqrt((X.astype(np.float64) ** 2).sum(1)).max()
    return err.max() / nrm, eps / nrm


@pytest.mark.parametrize("n,D,L", [(1, 4, 1), (127, 16, 5), (129, 20, 3), (1000, 64, 9), (4097, 100, 17),
                                   (20000, 128, 9), (33333, 256, 17), (5000, 256, 32), (3000, 13, 5),
                                   (3000, 300, 17), (70001, 32, 2)])
def test_projection_bound_random(ctx, n, D, L):
    rng = np.random.default_rng(n + D)
    X = (rng.standard_t(3, (n, D)) * rng.uniform(0.1, 10, D)).astype(np.float32)
    _check(ctx, X, _dirs(D, L, D))


@pytest.mark.parametrize("cfg,n", [(1, None), (2, 100_000), (3, 100_000), (4, 100_000), (5, 200_000)])
def test_projection_bound_configs(ctx, cfg, n):
    c = datagen.CONFIGS[cfg]
    X = datagen.generate_set(cfg, "A", n=n)
    D = X.shape[1]
    rel, bound = _check(ctx, X, _dirs(D, c.k + 1, cfg))
    print(f"cfg{cfg}: max |pi32 - pi64| / max||x|| = {rel:.2e} (bound {bound:.2e})")


def test_projection_variants_agree(ctx):
    """The tcgen05 and SIMT kernels both stay inside their own bounds on the same input."""
    rng = np.random.default_rng(3)
    X = rng.standard_normal((50_000, 256)).astype(np.float32)
    U = _dirs(256, 17, 7)
    tc = _check(ctx, X, U)
    from paper_2511_18207_b200 import option
    with option("k3_simt", 1):
        simt = _check(ctx, X, U)
    print(f"tcgen05 {tc[0]:.2e} (bound {tc[1]:.2e}); SIMT {simt[0]:.2e} (bound {simt[1]:.2e})")


def test_projection_special_values(ctx):
    rng = np.random.default_rng(11)
    X = rng.standard_normal((3000, 64)).astype(np.float32)
    X[:, 0] = 0.0
    X[::3, 1] = np.float32(-0.0)
    X[::7, 2] = np.float32(3e-40)  # subnormals
    X[17, 4] = np.float32(1e6)
    _check(ctx, X, _dirs(64, 9, 1))
