"""GPU parity for the NEXT rows of SURVEY.md §8(f).

f1 certified subset-full estimate: H^_sf against the oracle's subset_full on the same
   subsets, with its proven property H^_sf <= H (the exact undirected HD, also on GPU).
"""
import numpy as np
import pytest
import torch

import datagen
import oracle
from oracle import prohd as OP

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2511_18207_b200 import Context
    return Context(0)


def _tol_pair(X, Y, i, j):
    return 1e-5 * (float((X[i].astype(np.float64) ** 2).sum()) + float((Y[j].astype(np.float64) ** 2).sum()))


@pytest.mark.parametrize("cfg,n", [(1, None), (2, 20000), (4, 30000), (5, 65536)])
def test_certified_subset_full(ctx, cfg, n):
    c = datagen.CONFIGS[cfg]
    A, B = datagen.generate(cfg, n=n)
    m = c.m(A.shape[0])
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    g = ctx.prohd_estimate(At, Bt, c.k, m, return_indices=True, certified=True)
    ss = ctx.prohd_estimate(At, Bt, c.k, m, return_indices=True)
    assert np.array_equal(g["IA"], ss["IA"]) and np.array_equal(g["IB"], ss["IB"])  # same selection
    ref = OP.subset_full(A, B, g["IA"], g["IB"])
    assert abs(g["value"] - ref) <= 1e-4 * ref
    # witnesses: a in the subset, b the full-set nearest neighbour (fp64)
    assert g["ab"]["a"] in set(g["IA"].tolist()) and g["ba"]["a"] in set(g["IB"].tolist())
    rmin, arg = oracle.row_minima(A, B, rows=np.array([g["ab"]["a"]]))
    assert g["ab"]["b"] == int(arg[0]) and abs(g["ab"]["dist2"] - rmin[0]) <= 1e-12 * rmin[0]
    # provable: H^_sf <= H (exact), with the d2 tolerance of the two GPU computations
    H = ctx.hausdorff(At, Bt)
    tol = max(_tol_pair(A, B, H["ab"]["a"], H["ab"]["b"]), _tol_pair(B, A, H["ba"]["a"], H["ba"]["b"]))
    assert g["value"] ** 2 <= H["value"] ** 2 + tol
    # and H^_sf <= H^_ss is NOT implied; both are reported (cfg1 seed 0: H^_ss > H)
    if cfg == 1:
        assert ss["value"] > H["value"] >= g["value"]


# ---------------------------------------------------------------- f3: paper-literal parameters

@pytest.mark.parametrize("case", ["rc4", "rc64", "cfg2", "cfg4"])
def test_paper_literal_alpha(ctx, case):
    if case.startswith("rc"):
        D = int(case[2:])
        A, B = datagen.random_clouds(100_000, 100_000, D, seed=0)
    elif case == "cfg2":
        A, B = datagen.generate(2, n=50_000)
    else:
        A, B = datagen.generate(4, n=40_000)
    alpha = 0.01
    g = ctx.prohd_estimate_alpha(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), alpha,
                                 return_dirs=True, return_indices=True)
    ref = OP.estimate_paper(A, B, alpha)
    assert g["n_dirs"] == ref["n_dirs"] == ref["k"] + 1
    # selection with the GPU's directions (L3), then end to end (L5)
    D = A.shape[1]
    sel = []
    for X in (A, B):
        _, c0, c1 = OP.paper_parameters(D, alpha, X.shape[0])
        sel.append(OP.select_counts(X, g["U"], [c0] + [c1] * (g["U"].shape[1] - 1))["union"])
    assert np.array_equal(g["IA"], sel[0]) and np.array_equal(g["IB"], sel[1])
    assert np.array_equal(g["IA"], ref["IA"]) and np.array_equal(g["IB"], ref["IB"])
    assert abs(g["value"] - ref["value"]) <= 1e-4 * ref["value"]


# ---------------------------------------------------------------- f3: sampling baselines

@pytest.mark.parametrize("scheme", ["uniform", "systematic"])
def test_sampling_baselines(ctx, scheme):
    A, B = datagen.random_clouds(100_000, 80_000, 4, seed=1)
    alpha = 0.01
    if scheme == "uniform":  # ceil(alpha (nA + nB)) points from each set
        s = int(np.ceil(alpha * (A.shape[0] + B.shape[0])))
        ia, ib = datagen.uniform_sample(A.shape[0], s, 5), datagen.uniform_sample(B.shape[0], s, 6)
    else:  # permutation + every floor(1/alpha)-th point
        ia, ib = datagen.systematic_sample(A.shape[0], alpha, 5), datagen.systematic_sample(B.shape[0], alpha, 6)
    g = ctx.hausdorff_subsets(torch.from_numpy(A).cuda(), ia, torch.from_numpy(B).cuda(), ib)
    ref = OP.sampling_hd(A, B, ia, ib)
    assert abs(g["value"] - ref["value"]) <= 1e-4 * ref["value"]
    for side in ("ab", "ba"):
        X, Y = (A, B) if side == "ab" else (B, A)
        assert abs(g[side]["dist2"] - ref[side]["dist2"]) <= _tol_pair(X, Y, ref[side]["a"], ref[side]["b"])
    # host index lists and host points give the same answer
    h = ctx.hausdorff_subsets(torch.from_numpy(A), ia, torch.from_numpy(B), ib)
    assert h == g


# ---------------------------------------------------------------- f2: bound report

@pytest.mark.parametrize("cfg,n", [(1, None), (2, 20000), (3, 65536), (5, 65536)])
def test_bound_report(ctx, cfg, n):
    c = datagen.CONFIGS[cfg]
    A, B = datagen.generate(cfg, n=n)
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    e = ctx.prohd_estimate(At, Bt, c.k, c.m(A.shape[0]), return_dirs=True)
    U = e["U"]
    r = ctx.bounds(At, Bt, U)
    D = A.shape[1]
    mu = (A.astype(np.float64).sum(0) + B.astype(np.float64).sum(0)) / (A.shape[0] + B.shape[0])
    xmax = max(np.linalg.norm(A.astype(np.float64), axis=1).max(), np.linalg.norm(B.astype(np.float64), axis=1).max())
    g = (4 * D + 16) * 2.0 ** -24
    eps = (D + 8) * 2.0 ** -24 * xmax * 1.07
    for l in range(U.shape[1]):
        u = U[:, l]
        d0 = OP.delta(A, B, u)
        d1 = OP.delta(A, B, u, center=mu)
        # never below the exact value, and within the rounding-error inflation above it
        assert d0 <= r["delta_origin"][l] <= np.sqrt(d0 ** 2 + 2 * g * xmax ** 2) + 1e-12
        assert d1 <= r["delta_centered"][l] <= np.sqrt(d1 ** 2 + 2 * g * (xmax + np.linalg.norm(mu)) ** 2) + 1e-12
        hab, hba = OP.hd_1d(A.astype(np.float64) @ u, B.astype(np.float64) @ u)
        assert abs(r["hu_ab"][l] - hab) <= 2 * eps and abs(r["hu_ba"][l] - hba) <= 2 * eps
    HU = OP.multi_direction_hd(A, B, U)
    assert abs(r["H_U"] - HU) <= 2 * eps
    # Eq. (4): H_U <= H <= H_U + 2 min delta holds for the exact H (computed on the GPU)
    H = ctx.hausdorff(At, Bt)["value"]
    assert r["H_U"] <= H * (1 + 1e-6) + 2 * eps
    assert H <= r["upper"] + 1e-6 * H
