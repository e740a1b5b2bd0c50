"""The sharded-ProHD phase calls on one GPU: G row shards simulated in sequence (the sums,
concatenations and maxima stand in for the NCCL collectives), compared with the one-shot
prohd_estimate and with the oracle. Also: exact HD via directed_hd_local on row shards is
bit-identical to the unsharded call (GPU-count invariance of the packed key)."""
import numpy as np
import pytest
import torch

import datagen
from oracle import prohd as OP
from paper_2511_18207_b200.dist import CudaPhases, row_range, unpack_key

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2511_18207_b200 import Context
    return Context(0)


def _sim_sharded(ctx, A, B, k, m, G, dmma=True):
    ph = CudaPhases(ctx, dmma=dmma)
    nA, nB, D = A.shape[0], B.shape[0], A.shape[1]
    la = [row_range(nA, g, G) for g in range(G)]
    lb = [row_range(nB, g, G) for g in range(G)]
    s = ph.shift(A[:4096], B[:4096])
    # C0: MAX over the shards' column ranges (int8 Gram), C1: SUM of the moments
    colmax = None
    for g in range(G):
        cm = ph.local_colmax(A[la[g][0]:la[g][1]], B[lb[g][0]:lb[g][1]], s)
        if cm is not None:
            colmax = cm if colmax is None else torch.maximum(colmax, cm)
    mom = None
    for g in range(G):
        part = ph.local_moments(A[la[g][0]:la[g][1]], B[lb[g][0]:lb[g][1]], s, colmax)
        mom = part if mom is None else mom + part
    dirs, nd = ph.directions(mom, nA, nB, D, k, s)
    unions, subsets = [], []
    for X, rng in ((A, la), (B, lb)):
        lists = [ph.local_candidates(X[lo:hi], lo, dirs, m) for lo, hi in rng]
        union = ph.merge_union(torch.stack([v for v, _ in lists]), torch.stack([i for _, i in lists]), m,
                               X.shape[0])
        rows = torch.cat([ph.gather_owned(X[lo:hi], lo, union)[0] for lo, hi in rng])
        unions.append(union)
        subsets.append(rows)
    out = {}
    centre = ctx.centre(subsets[0], subsets[1])  # prohd_estimate's subset-HD centre
    for side, (R, Cm, uR, uC) in {"ab": (subsets[0], subsets[1], unions[0], unions[1]),
                                  "ba": (subsets[1], subsets[0], unions[1], unions[0])}.items():
        keys = []
        for g in range(G):
            lo, hi = row_range(R.shape[0], g, G)
            if hi > lo:
                keys.append(ctx.directed_hd_local(R[lo:hi], lo, Cm, centre))
        key = max(keys)
        _, row = unpack_key(key)
        w = ctx.directed_hd_witness(R[row], Cm)
        out[side] = {"a": int(uR[row]), "b": int(uC[w["b"]]), "dist2": w["dist2"]}
    value = float(np.sqrt(max(out["ab"]["dist2"], out["ba"]["dist2"])))
    return {"value": value, "IA": unions[0].cpu().numpy(), "IB": unions[1].cpu().numpy(), "U": dirs.cpu().numpy(),
            "n_dirs": nd, **out}


@pytest.mark.parametrize("cfg,n,G", [(1, None, 2), (2, 20000, 3), (5, 65536, 2), (4, 65536, 4)])
def test_sharded_phases_equal_single(ctx, cfg, n, G):
    c = datagen.CONFIGS[cfg]
    A, B = datagen.generate(cfg, n=n)
    m = c.m(A.shape[0])
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    # the sharded moments phase keeps the fp64 DMMA Gram (its shift is fixed across ranks): compare
    # against the one-shot call on the same Gram path, bit for bit
    from paper_2511_18207_b200 import option
    with option("k1_path", 0):
        one = ctx.prohd_estimate(At, Bt, c.k, m, return_dirs=True, return_indices=True)
    sh = _sim_sharded(ctx, At, Bt, c.k, m, G)
    assert sh["n_dirs"] == one["n_dirs"]
    assert np.allclose(sh["U"].T, one["U"], rtol=0, atol=1e-12)
    assert np.array_equal(sh["IA"], one["IA"]) and np.array_equal(sh["IB"], one["IB"])
    assert sh["value"] == one["value"]
    assert (sh["ab"]["a"], sh["ab"]["b"]) == (one["ab"]["a"], one["ab"]["b"])
    assert (sh["ba"]["a"], sh["ba"]["b"]) == (one["ba"]["a"], one["ba"]["b"])
    ref = OP.estimate(A, B, c.k, m)
    assert np.array_equal(sh["IA"], ref["IA"]) and np.array_equal(sh["IB"], ref["IB"])


@pytest.mark.parametrize("G", [2, 3, 8])
def test_exact_key_invariant_to_shard_count(ctx, G):
    A, B = datagen.generate(2, n=30000)
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    one = ctx.directed_hd(At, Bt)
    keys = []
    for g in range(G):
        lo, hi = row_range(A.shape[0], g, G)
        keys.append(ctx.directed_hd_local(At[lo:hi], lo, Bt))
    key = max(keys)
    d2, row = unpack_key(key)
    assert row == one["a"] and np.float32(d2) == np.float32(one["dist2_tc"])
    w = ctx.directed_hd_witness(At[row], Bt)
    assert w["b"] == one["b"] and w["dist2"] == one["dist2"]


@pytest.mark.parametrize("cfg,n,G", [(1, None, 2), (3, 30000, 3), (5, 65536, 4), (4, 40000, 8)])
def test_sharded_int8_moments(ctx, cfg, n, G):
    """The sharded moments on the int8 Gram (prohd_local_colmax -> MAX -> prohd_local_moments_i8
    -> SUM): every shard quantises on the grid of the global column maxima, the grid the one-shot
    call picks, so the directions agree with the one-shot int8 call to fp64 rounding and the
    selections, subsets and estimate are identical (and equal the oracle's)."""
    c = datagen.CONFIGS[cfg]
    A, B = datagen.generate(cfg, n=n)
    m = c.m(A.shape[0])
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    one = ctx.prohd_estimate(At, Bt, c.k, m, return_dirs=True, return_indices=True)
    sh = _sim_sharded(ctx, At, Bt, c.k, m, G, dmma=False)
    assert sh["n_dirs"] == one["n_dirs"]
    assert np.allclose(sh["U"].T, one["U"], rtol=0, atol=1e-9)
    assert np.array_equal(sh["IA"], one["IA"]) and np.array_equal(sh["IB"], one["IB"])
    assert sh["value"] == one["value"]
    ref = OP.estimate(A, B, c.k, m)
    assert np.array_equal(sh["IA"], ref["IA"]) and np.array_equal(sh["IB"], ref["IB"])


def test_sharded_int8_empty_set_shard(ctx):
    """A shard holding rows of one set only (nB_local = 0) and an empty shard: the int8 phase
    calls accept them and the summed moments match the one-shot covariance path."""
    rng = np.random.default_rng(5)
    D = 64
    A = rng.standard_normal((3000, D)).astype(np.float32)
    B = (rng.standard_normal((2000, D)) + 0.5).astype(np.float32)
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    ph = CudaPhases(ctx, dmma=False)
    s = ph.shift(At[:4096], Bt[:4096])
    shards = [(At[:1000], Bt[:0]), (At[1000:3000], Bt[:2000]), (At[:0], Bt[:0])]
    colmax = None
    for a_, b_ in shards:
        cm = ph.local_colmax(a_, b_, s)
        colmax = cm if colmax is None else torch.maximum(colmax, cm)
    mom = sum(ph.local_moments(a_, b_, s, colmax) for a_, b_ in shards)
    X = np.concatenate([A, B]).astype(np.float64) - s
    G = X.T @ X
    Gd = mom[2 * D:].cpu().numpy().reshape(D, D)
    scale = np.abs(X).max(0)
    assert np.all(np.abs(Gd - G) <= 2.0 ** -26 * X.shape[0] * np.outer(scale, scale))
    assert np.allclose(mom[:D].cpu().numpy(), (np.asarray(A, np.float64) - s).sum(0), rtol=0,
                       atol=1e-6 * 3000 * scale.max())
