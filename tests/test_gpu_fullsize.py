"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

Exact HD: the full-size directed HD runs on the GPU; the fp64
oracle checks a seeded sample of rows of A against ALL of B (plus the GPU's witness
row), because the whole oracle problem takes hours on the host (the sample sizes
below keep each case within ~1 minute of host time):
  * every sampled row minimum within the Q17 tolerance of the oracle's;
  * the reported value equals the oracle's fp64 minimum of the reported witness row,
    and the witness column is that row's oracle nearest neighbour;
  * no sampled row's oracle minimum exceeds the reported value (beyond tolerance).
ProHD: the oracle runs Alg. 3 in full at these sizes; layers L2/L3/L5 as in
test_gpu_prohd.py.
"""
import numpy as np
import pytest
import torch

import datagen
import oracle
from oracle import prohd as OP

pytestmark = pytest.mark.gpu

ROWS = {3: 2000, 4: 600, 5: 400}


@pytest.fixture(scope="module")
def ctx():
    from paper_2511_18207_b200 import Context
    return Context(0)


@pytest.mark.parametrize("cfg", [3, 4, 5])
def test_exact_full_size_sampled(ctx, cfg):
    A = datagen.generate_set(cfg, "A")
    B = datagen.generate_set(cfg, "B")
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    r = ctx.directed_hd(At, Bt)
    rm = ctx.directed_hd_rowmin(At, Bt).cpu().numpy()
    rows = np.union1d(datagen.sample_rows(A.shape[0], ROWS[cfg], seed=cfg), [r["a"]])
    ref, arg = oracle.row_minima(A, B, rows=rows)
    na = (A[rows].astype(np.float64) ** 2).sum(1)
    nb = (B[arg].astype(np.float64) ** 2).sum(1)
    err = np.abs(rm[rows].astype(np.float64) - ref) / (na + nb)
    assert err.max() <= 1e-5, f"row-min rel err {err.max():.2e}"
    w = int(np.searchsorted(rows, r["a"]))
    assert r["b"] == int(arg[w])
    assert abs(r["dist2"] - ref[w]) <= 1e-12 * ref[w]
    tol = 1e-5 * (na.max() + nb.max())
    assert ref.max() <= r["dist2"] + tol
    # the reported row is the GPU's argmax of its own row minima
    assert rm.max() == np.float32(r["dist2_tc"])


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_prohd_full_size(ctx, cfg):
    c = datagen.CONFIGS[cfg]
    A = datagen.generate_set(cfg, "A")
    B = datagen.generate_set(cfg, "B")
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    g = ctx.prohd_estimate(At, Bt, c.k, c.m(), return_dirs=True, return_indices=True)
    U = g["U"]
    ref = OP.estimate(A, B, c.k, c.m())
    # L2
    assert np.linalg.norm(U[:, 0] - ref["u0"]) <= 1e-9
    C = ref["C"]
    cn = np.linalg.norm(C, 2)
    for l in range(1, U.shape[1]):
        v = U[:, l]
        assert np.linalg.norm(C @ v - (v @ C @ v) * v) <= 1e-9 * cn
    # L3: oracle selection with the GPU's directions -> identical unions
    sA = OP.select(A, U, c.m())
    sB = OP.select(B, U, c.m())
    assert np.array_equal(g["IA"], sA["union"]) and np.array_equal(g["IB"], sB["union"])
    # L4/L5: identical subsets (also vs the oracle's own directions) -> H^ within 1e-4
    assert np.array_equal(g["IA"], ref["IA"]) and np.array_equal(g["IB"], ref["IB"])
    assert abs(g["value"] - ref["value"]) <= 1e-4 * ref["value"]
    assert (g["size_a"], g["size_b"]) == (ref["size_a"], ref["size_b"])
