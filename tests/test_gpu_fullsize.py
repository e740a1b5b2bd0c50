"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

Exact HD (BASELINE.json cfg5 "checks exact HD on 20,000 random A-rows
against all of B"): the full-size directed HD runs on the GPU; the fp64 oracle checks 20,000
seeded rows of A against ALL of B (plus the GPU's witness row), because the whole oracle
problem takes hours on the host (cfg5: ~5 min of host time at ~0.12 Gpair/s on 16 cores):
  * every sampled row minimum within the Q17 tolerance of the oracle's;
  * the reported value equals the oracle's fp64 minimum of the reported witness row,
    and the witness column is that row's oracle nearest neighbour;
  * no sampled row's oracle minimum exceeds the reported value (beyond tolerance).
Undirected H at full size through hausdorff_minima (the hausdorff() sweep:
fused bidirectional at D >= 128): 2,000 sampled rows of A (row minima; the directed test above
covers 20,000) and 4,000 sampled rows of B (the fused sweep's column minima) against all of the other set, with the same checks per
direction and the reported H = the larger side's fp64 witness distance.
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

ROWS = {3: 20000, 4: 20000, 5: 20000}
COLS = {3: 4000, 4: 4000, 5: 4000}
UROWS = {3: 2000, 4: 2000, 5: 2000}  # A side of the undirected check (the directed test covers 20,000)


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


def _check_side(X, Y, mins, rows, wit):
    """Sampled rows of X (and the witness row) against all of Y: Q17 per row, witness, max."""
    rows = np.union1d(rows, [wit["a"]])
    ref, arg = oracle.row_minima(X, Y, rows=rows)
    nx = (X[rows].astype(np.float64) ** 2).sum(1)
    ny = (Y[arg].astype(np.float64) ** 2).sum(1)
    err = np.abs(mins[rows].astype(np.float64) - ref) / (nx + ny)
    assert err.max() <= 1e-5, f"row-min rel err {err.max():.2e}"
    w = int(np.searchsorted(rows, wit["a"]))
    assert wit["b"] == int(arg[w])
    assert abs(wit["dist2"] - ref[w]) <= 1e-12 * ref[w]
    assert ref.max() <= wit["dist2"] + 1e-5 * (nx.max() + ny.max())
    assert mins.max() == np.float32(wit["dist2_tc"])
    return err.max()


@pytest.mark.parametrize("cfg", [3, 4, 5])
def test_undirected_full_size_sampled(ctx, cfg):
    A = datagen.generate_set(cfg, "A")
    B = datagen.generate_set(cfg, "B")
    h, rm, cm = ctx.hausdorff_minima(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
    rm, cm = rm.cpu().numpy(), cm.cpu().numpy()
    e1 = _check_side(A, B, rm, datagen.sample_rows(A.shape[0], UROWS[cfg], seed=cfg + 10), h["ab"])
    e2 = _check_side(B, A, cm, datagen.sample_rows(B.shape[0], COLS[cfg], seed=cfg + 20), h["ba"])
    side = h["ab"] if h["ab"]["dist2"] >= h["ba"]["dist2"] else h["ba"]
    assert h["value"] == side["dist"]
    print(f"cfg{cfg}: H={h['value']:.6f}; max row-min err / Q17: A->B {e1 / 1e-5:.3f}, B->A {e2 / 1e-5:.3f}")


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
    _, Cg, path = ctx.covariance(At, Bt)
    tol = max(1e-9 * cn, 2.0 * np.linalg.norm(Cg - C, 2) + 1e-11 * cn)  # see test_gpu_prohd._direction_tol
    for l in range(1, U.shape[1]):
        v = U[:, l]
        assert np.linalg.norm(C @ v - (v @ C @ v) * v) <= tol
    print(f"cfg{cfg}: Gram path {'int8' if path else 'fp64 DMMA'}, ||C_gpu - C||_2 / ||C|| = "
          f"{np.linalg.norm(Cg - C, 2) / cn:.2e}")
    # L3: oracle selection with the GPU's directions -> identical unions
    sA = OP.select(A, U, c.m())
    sB = OP.select(B, U, c.m())
    assert np.array_equal(g["IA"], sA["union"]) and np.array_equal(g["IB"], sB["union"])
    # L4/L5: identical subsets (also vs the oracle's own directions) -> H^ within 1e-4
    assert np.array_equal(g["IA"], ref["IA"]) and np.array_equal(g["IB"], ref["IB"])
    assert abs(g["value"] - ref["value"]) <= 1e-4 * ref["value"]
    assert (g["size_a"], g["size_b"]) == (ref["size_a"], ref["size_b"])
