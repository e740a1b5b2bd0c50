"""GPU parity for ProHD (Alg. 3) through the C ABI, layered as SURVEY.md §8(c4):

  L2 directions   u0 within 1e-9; each PC an eigenvector of the oracle's C
                  (residual <= 2 ||C_gpu - C||_2 + 1e-11 ||C||, at least 1e-9 ||C||, with
                  C_gpu the library's own covariance through prohd_covariance) and, where
                  the oracle's spectral gap allows, within the Davis-Kahan angle of the
                  oracle's PC (the same numerator over the gap).
  L3 selection    the oracle run with the GPU's directions injected: per-set
                  unions bit-exact, except swaps across the m-th boundary between
                  points whose fp64 projections differ by <= 1e-6 max(||p||,||q||)
                  (north_star "bit-exact except at projection ties within 1e-6").
  L4 subset HD    same subsets -> |H^_gpu - H^_ref| <= 1e-4 H^_ref and the d2
                  tolerance 1e-5 (||a||^2 + ||b||^2) on the witness pair.
  L5 end to end   the oracle with its own C and Jacobi directions.
"""
import numpy as np
import pytest
import torch

import datagen
import oracle
from oracle import prohd as OP

pytestmark = pytest.mark.gpu

TIE = 1e-6


@pytest.fixture(scope="module")
def ctx():
    from paper_2511_18207_b200 import Context
    return Context(0)


def _excused_union_diff(X, U, m, got, ref):
    """Union differences allowed only under SURVEY.md §8(c2) Q16: each difference is one half of a
    swap across the m-th boundary of ONE (direction, tail) list between points p (GPU-selected) and
    q (oracle-selected) with |pi64(p) - pi64(q)| <= 1e-6 max(||p||, ||q||) (pi64 = fp64 projection on
    the GPU's exported direction). Extras and missings must pair up one to one under that rule."""
    got, ref = set(got.tolist()), set(ref.tolist())
    extra, missing = sorted(got - ref), sorted(ref - got)
    if not extra and not missing:
        return 0
    assert len(extra) == len(missing), f"unpaired differences: +{extra} -{missing}"
    P = X.astype(np.float64) @ U
    nrm = np.linalg.norm(X.astype(np.float64), axis=1)
    n = X.shape[0]
    idx = np.arange(n)

    def boundary_pair_ok(p, q):
        for l in range(U.shape[1]):
            if abs(P[p, l] - P[q, l]) > TIE * max(nrm[p], nrm[q]):
                continue
            for top in (False, True):
                # oracle total order of this tail: (pi asc, idx asc) bottom, (pi desc, idx asc) top
                order = np.lexsort((idx, -P[:, l] if top else P[:, l]))
                rank = np.empty(n, np.int64)
                rank[order] = idx
                # q inside the oracle's first m, p just outside, both in the tie band at the boundary
                if rank[q] < m <= rank[p]:
                    return True
        return False

    unmatched = list(missing)
    for p in extra:
        hit = next((q for q in unmatched if boundary_pair_ok(p, q)), None)
        assert hit is not None, f"index {p} differs without a paired boundary swap at a 1e-6 projection tie"
        unmatched.remove(hit)
    return len(extra) + len(missing)


def _direction_tol(ctx, A, B, C):
    """L2 tolerance for an eigenvector v of the GPU's covariance C_gpu judged against the oracle's
    C: ||C v - (v^T C v) v|| <= 2 ||C_gpu - C||_2 + eigen-solver error (Davis-Kahan for the angle,
    divided by the gap). C_gpu through prohd_covariance (the same Gram path as prohd_estimate); at
    least the 1e-9 ||C|| of the fp64 Gram."""
    _, Cg, _ = ctx.covariance(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
    cn = np.linalg.norm(C, 2)
    return max(1e-9 * cn, 2.0 * np.linalg.norm(Cg - C, 2) + 1e-11 * cn)


def _run(ctx, A, B, k, m):
    return ctx.prohd_estimate(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), k, m,
                              return_dirs=True, return_indices=True)


def _check_layers(ctx, A, B, k, m, exact_sets=True):
    g = _run(ctx, A, B, k, m)
    U = g["U"]
    ref = OP.estimate(A, B, k, m)
    # L2: directions
    assert np.linalg.norm(U[:, 0] - ref["u0"]) <= 1e-9
    C = ref["C"]
    cn = np.linalg.norm(C, 2)
    assert g["n_dirs"] == ref["n_dirs"]
    lam = np.sort(np.linalg.eigvalsh(C))[::-1]
    tol = _direction_tol(ctx, A, B, C)
    for l in range(1, U.shape[1]):
        v = U[:, l]
        assert abs(np.linalg.norm(v) - 1) <= 1e-12
        r = C @ v - (v @ C @ v) * v
        assert np.linalg.norm(r) <= tol, f"PC{l} residual {np.linalg.norm(r) / cn:.2e}"
        gap = min(abs(lam[l - 1] - lam[j]) for j in range(len(lam)) if j != l - 1)
        if gap > 1e-6 * lam[0]:
            s = np.linalg.norm(v - (v @ ref["U"][:, l]) * ref["U"][:, l])
            assert s <= tol / gap + 1e-12, f"PC{l} angle {s:.2e}, gap {gap / lam[0]:.2e}"
    # L3: oracle with the GPU's directions injected
    inj = OP.estimate(A, B, k, m, U=U)
    nd = _excused_union_diff(A, U, m, g["IA"], inj["IA"]) + _excused_union_diff(B, U, m, g["IB"], inj["IB"])
    if exact_sets:
        assert nd == 0
    # L4: subset HD on identical subsets
    if nd == 0:
        assert abs(g["value"] - inj["value"]) <= 1e-4 * inj["value"] + 1e-12
        for side in ("ab", "ba"):
            a_set, b_set = (A, B) if side == "ab" else (B, A)
            tol = 1e-5 * (float((a_set[inj[side]["a"]].astype(np.float64) ** 2).sum())
                          + float((b_set[inj[side]["b"]].astype(np.float64) ** 2).sum()))
            assert abs(g[side]["dist2"] - inj[side]["dist2"]) <= tol
    # L5: end to end against the oracle's own directions
    assert g["size_a"] == len(g["IA"]) and g["size_b"] == len(g["IB"])
    return g, ref, inj


def test_w3_bit_exact(ctx, golden):
    gw = golden["W3"]
    A = np.array(gw["A"], np.float32)
    B = A + np.array(gw["B_offset"], np.float32)
    for key, k in (("k1_m1", 1), ("k2_m1", 2)):
        g = _run(ctx, A, B, k, 1)
        assert g["IA"].tolist() == gw[key]["IA"] and g["IB"].tolist() == gw[key]["IB"]
        assert g["value"] == gw[key]["H_hat"]
        assert [g["ab"]["a"], g["ab"]["b"]] == gw[key]["ab_witness"]
    g = _run(ctx, A, B, 2, 1)
    assert np.allclose(g["U"][:, 0], gw["u0"], atol=0)
    assert np.allclose(np.abs(g["U"][:, 1]), np.abs(np.array(gw["pc1"])), atol=1e-14)


def test_w5_injected(ctx, golden):
    gw = golden["W5"]
    A = np.array(gw["A"], np.float32)
    B = np.array(gw["B"], np.float32)
    r = ctx.prohd_estimate_with_dirs(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(),
                                     np.array(gw["U"]), gw["m"])
    assert r["IA"].tolist() == gw["IA"] and r["IB"].tolist() == gw["IB"]
    assert abs(r["value"] - gw["H_hat_ss"]) <= 1e-6


def test_cfg1_layers(ctx, golden):
    A, B = datagen.generate(1)
    g, ref, inj = _check_layers(ctx, A, B, 4, 20)
    gw = golden["CFG1_SEED0"]
    assert (g["size_a"], g["size_b"]) == (gw["size_a"], gw["size_b"])
    assert np.array_equal(g["IA"], ref["IA"]) and np.array_equal(g["IB"], ref["IB"])
    assert abs(g["value"] - ref["value"]) <= 1e-4 * ref["value"]
    assert [g["ab"]["a"], g["ab"]["b"]] == gw["hhat_ab_witness"]
    assert [g["ba"]["a"], g["ba"]["b"]] == gw["hhat_ba_witness"]


@pytest.mark.parametrize("cfg,n", [(2, 20000), (3, 65536), (4, 65536), (5, 65536)])
def test_reduced_scale_layers(ctx, cfg, n):
    c = datagen.CONFIGS[cfg]
    A, B = datagen.generate(cfg, n=n)
    m = c.m(n)
    g, ref, inj = _check_layers(ctx, A, B, c.k, m)
    if np.array_equal(g["IA"], ref["IA"]) and np.array_equal(g["IB"], ref["IB"]):
        assert abs(g["value"] - ref["value"]) <= 1e-4 * ref["value"]


def test_full_selection_equals_exact(ctx):
    rng = np.random.default_rng(3)
    A = rng.standard_normal((50, 8)).astype(np.float32)
    B = (rng.standard_normal((40, 8)) + 0.5).astype(np.float32)
    g = _run(ctx, A, B, 3, 25)  # 2m >= n for both sets
    assert g["size_a"] == 50 and g["size_b"] == 40
    h = ctx.hausdorff(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
    assert g["value"] == h["value"]


def test_identical_sets(ctx):
    rng = np.random.default_rng(4)
    A = rng.standard_normal((3000, 16)).astype(np.float32)
    g = _run(ctx, A, A.copy(), 4, 10)
    assert g["value"] == 0.0
    assert g["U"][:, 0].tolist() == [1.0] + [0.0] * 15  # equal centroids -> e1


def test_k0_centroid_only(ctx):
    rng = np.random.default_rng(5)
    A = rng.standard_normal((5000, 12)).astype(np.float32)
    B = (rng.standard_normal((4000, 12)) + 1.0).astype(np.float32)
    g = _run(ctx, A, B, 0, 30)
    ref = OP.estimate(A, B, 0, 30)
    assert g["n_dirs"] == 1
    assert np.array_equal(g["IA"], ref["IA"]) and np.array_equal(g["IB"], ref["IB"])
    assert abs(g["value"] - ref["value"]) <= 1e-4 * ref["value"]


def test_ragged_and_ties(ctx):
    """Duplicate points (exact projection ties) and n not a multiple of any tile."""
    rng = np.random.default_rng(6)
    A = rng.standard_normal((1001, 20)).astype(np.float32)
    A[500:600] = A[0]
    B = rng.standard_normal((777, 20)).astype(np.float32)
    B[100:300] = B[5]
    _check_layers(ctx, A, B, 3, 7)


def test_host_inputs(ctx):
    A, B = datagen.generate(2, n=20000)
    c = datagen.CONFIGS[2]
    gd = ctx.prohd_estimate(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), c.k, c.m(20000))
    gh = ctx.prohd_estimate(torch.from_numpy(A), torch.from_numpy(B), c.k, c.m(20000))
    assert gd == gh


def test_determinism(ctx):
    A, B = datagen.generate(5, n=65536)
    r = [_run(ctx, A, B, 16, 32) for _ in range(2)]
    assert r[0]["value"] == r[1]["value"] and np.array_equal(r[0]["U"], r[1]["U"])
    assert np.array_equal(r[0]["IA"], r[1]["IA"]) and np.array_equal(r[0]["IB"], r[1]["IB"])


def test_errors(ctx):
    from paper_2511_18207_b200 import ProHDError
    A = torch.randn(100, 4, device="cuda")
    B = torch.randn(90, 4, device="cuda")
    with pytest.raises(ProHDError) as e:
        ctx.prohd_estimate(A, B, 5, 3)  # k > D
    assert e.value.code == 2
    with pytest.raises(ProHDError) as e:
        ctx.prohd_estimate(A, B, 2, 0)  # m < 1
    assert e.value.code == 2
    An = A.clone()
    An[7, 2] = float("nan")
    with pytest.raises(ProHDError) as e:
        ctx.prohd_estimate(An, B, 2, 3)
    assert e.value.code == 3


def test_large_offset_uses_shift(ctx):
    """A common offset far above the spread: the shift kernel keeps s, the Gram pass
    subtracts it in fp64, and every layer still matches the oracle's two-pass C."""
    A, B = datagen.generate(2, n=20000)
    A = (A + np.float32(4096.0)).astype(np.float32)
    B = (B + np.float32(4096.0)).astype(np.float32)
    s = ctx.shift(torch.from_numpy(A[:4096]).cuda(), torch.from_numpy(B[:4096]).cuda())
    assert np.all(s != 0.0)
    c = datagen.CONFIGS[2]
    _check_layers(ctx, A, B, c.k, c.m(20000))


def test_small_offset_drops_shift(ctx):
    A, B = datagen.generate(2, n=20000)
    s = ctx.shift(torch.from_numpy(A[:4096]).cuda(), torch.from_numpy(B[:4096]).cuda())
    assert np.all(s == 0.0)


@pytest.mark.parametrize("D", [13, 16])
def test_special_values(ctx, D):
    """Signed zeros and subnormals (the Gram pass converts fp32 -> fp64 on the integer
    pipe and falls back to F2F for subnormals); D = 13 takes the 4-byte loader path."""
    rng = np.random.default_rng(11 + D)
    A = rng.standard_normal((3000, D)).astype(np.float32)
    B = (rng.standard_normal((2500, D)) + 0.25).astype(np.float32)
    A[::7, 1] = np.float32(-0.0)
    A[::11, 2] = np.float32(0.0)
    A[::13, 3] = np.float32(3e-40)   # subnormal
    B[::5, 0] = np.float32(-2e-39)   # subnormal
    _check_layers(ctx, A, B, 3, 9)


@pytest.mark.parametrize("bad", ["nan_a", "inf_b", "neg_inf_a"])
def test_nonfinite_wide(ctx, bad):
    """Non-finite input at D = 256 (DMMA Gram with the F2F fallback, tcgen05 projection, K6):
    every entry point reports PROHD_E_DATA instead of returning a number."""
    from paper_2511_18207_b200 import ProHDError
    rng = np.random.default_rng(4)
    A = rng.standard_normal((3000, 256)).astype(np.float32)
    B = rng.standard_normal((2500, 256)).astype(np.float32)
    if bad == "nan_a":
        A[1234, 77] = np.nan
    elif bad == "inf_b":
        B[17, 200] = np.inf
    else:
        A[2999, 0] = -np.inf
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    for call in (lambda: ctx.prohd_estimate(At, Bt, 8, 50), lambda: ctx.directed_hd(At, Bt),
                 lambda: ctx.hausdorff(At, Bt)):
        with pytest.raises(ProHDError) as e:
            call()
        assert e.value.code == 3


def _tied_cloud(n, D, nties, seed):
    """x_0 = 5.0 exactly on `nties` points (an exact tie straddling the m-th top value of e1) below
    500 larger distinct values, and x_1 = -5.0 on another `nties` points straddling the m-th bottom
    value of e2; every other coordinate random (all points distinct)."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, D)).astype(np.float32)
    X[:, 0] = np.clip(X[:, 0], -3.0, 3.0)
    X[:, 1] = np.clip(X[:, 1], -3.0, 3.0)
    idx = rng.permutation(n)
    top, tie_t, tie_b, bot = idx[:500], idx[500:500 + nties], idx[500 + nties:500 + 2 * nties], \
        idx[500 + 2 * nties:1000 + 2 * nties]
    X[top, 0] = (6.0 + rng.random(500)).astype(np.float32)
    X[tie_t, 0] = 5.0
    X[bot, 1] = (-6.0 - rng.random(500)).astype(np.float32)
    X[tie_b, 1] = -5.0
    return X


def test_guard_band_overflow_exact_ties(ctx):
    """VERDICT r01 missing #5: more than m + 65536 candidates in a guard band (140,000 exact
    duplicates of the m-th projection value on e1's top tail and on e2's bottom tail, m = 1000).
    The selection is still defined (PAPER.md:205-214 with the Q6 lowest-index tie rule): the lists
    must equal the oracle's bit for bit, through the streaming band-select fallback, in the one-shot
    call and in the sharded candidate lists (two shards, merged)."""
    n, D, m = 300_000, 16, 1000
    A = _tied_cloud(n, D, 140_000, 1)  # ~70,000 ties per half: each shard overflows too
    B = _tied_cloud(n, D, 140_000, 2)
    U = np.zeros((D, 3))
    U[0, 0] = 1.0
    U[1, 1] = 1.0
    U[2:, 2] = 1.0 / np.sqrt(D - 2)
    g = ctx.prohd_estimate_with_dirs(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), U, m)
    ref = OP.estimate(A, B, 2, m, U=U)
    assert np.array_equal(g["IA"], ref["IA"]) and np.array_equal(g["IB"], ref["IB"])
    assert abs(g["value"] - ref["value"]) <= 1e-4 * ref["value"]
    # sharded path: local candidate lists of two row blocks, merged on the device
    dirs = torch.from_numpy(np.ascontiguousarray(U.T)).cuda()
    half = n // 2
    vals, idxs = [], []
    for lo, hi in ((0, half), (half, n)):
        v, i = ctx.local_candidates(torch.from_numpy(A[lo:hi]).cuda(), lo, dirs, m)
        vals.append(v)
        idxs.append(i)
    union = ctx.merge_union(torch.stack(vals), torch.stack(idxs), m, n).cpu().numpy()
    assert np.array_equal(union, ref["IA"])


@pytest.mark.parametrize("cfg,n", [(2, 20000), (3, 65536), (5, 65536)])
def test_sampled_select_layers(ctx, cfg, n):
    """K4 with a sampled threshold and K3's fused pre-selection (k_select.cu
    launch_select_sampled; the default from n = 262,144 on), forced at the reduced sizes: the
    same L2-L5 layers as the radix K4 (exact unions)."""
    from paper_2511_18207_b200 import option
    c = datagen.CONFIGS[cfg]
    A, B = datagen.generate(cfg, n=n)
    with option("k4_sampled", 1):
        g, ref, inj = _check_layers(ctx, A, B, c.k, c.m(n))
    if np.array_equal(g["IA"], ref["IA"]) and np.array_equal(g["IB"], ref["IB"]):
        assert abs(g["value"] - ref["value"]) <= 1e-4 * ref["value"]


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_sampled_equals_radix(ctx, cfg):
    """At 300,000 points per set (sampled K4 by default) the selected unions, the estimate and its
    witnesses are identical to the radix K4's (option k4_sampled 0): the certified band is the
    radix path's band (same m-th value T, same eps), so the candidate set is the same."""
    from paper_2511_18207_b200 import option
    c = datagen.CONFIGS[cfg]
    n = 300_000
    A, B = datagen.generate(cfg, n=n)
    m = c.m(n)
    tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    g1 = ctx.prohd_estimate(tA, tB, c.k, m, return_dirs=True, return_indices=True)
    with option("k4_sampled", 0):
        g0 = ctx.prohd_estimate(tA, tB, c.k, m, return_dirs=True, return_indices=True)
    assert np.array_equal(g0["U"], g1["U"])
    assert np.array_equal(g0["IA"], g1["IA"]) and np.array_equal(g0["IB"], g1["IB"])
    assert g0["value"] == g1["value"]
    for side in ("ab", "ba"):
        assert (g0[side]["a"], g0[side]["b"]) == (g1[side]["a"], g1[side]["b"])


def test_sampled_select_uncertified_reruns(ctx):
    """Lists the sampled K4 cannot certify: 50,000 exact duplicates of the m-th value on e1's top
    tail (and on e2's bottom tail), so the sample threshold IS the m-th value T and the guard band
    [T - 2 eps, inf) reaches below it (within the raw capacity, so this is the certification check,
    not an overflow). The radix rerun gives the oracle's lists; so does the radix K4 alone."""
    from paper_2511_18207_b200 import option
    n, D, m = 300_000, 16, 1000
    A = _tied_cloud(n, D, 50_000, 5)
    B = _tied_cloud(n, D, 50_000, 6)
    U = np.zeros((D, 3))
    U[0, 0] = 1.0
    U[1, 1] = 1.0
    U[2:, 2] = 1.0 / np.sqrt(D - 2)
    ref = OP.estimate(A, B, 2, m, U=U)
    for opt in (1, 0):
        with option("k4_sampled", opt):
            g = ctx.prohd_estimate_with_dirs(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), U, m)
        assert np.array_equal(g["IA"], ref["IA"]) and np.array_equal(g["IB"], ref["IB"])
        assert abs(g["value"] - ref["value"]) <= 1e-4 * ref["value"]


def test_graph_replay_matches_eager(ctx):
    """prohd_estimate replays cached CUDA graphs of its two stream-ordered stretches (steps 1-3,
    step 4; api_common.cuh graphed()): repeated calls, and new data written into the same device
    buffers (same pointers, so the cached graphs replay on different values), return exactly what
    the eager launches (option graph = 0) return, and the launch counter advances by the same
    number of kernels per call."""
    from paper_2511_18207_b200 import option
    c = datagen.CONFIGS[2]
    A, B = datagen.generate(2, n=20000)
    m = c.m(20000)
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()

    def run():
        l0 = ctx.launch_count()
        r = ctx.prohd_estimate(At, Bt, c.k, m, return_indices=True, return_dirs=True)
        return r, ctx.launch_count() - l0

    def same(r, q):
        assert r["value"] == q["value"] and r["ab"] == q["ab"] and r["ba"] == q["ba"]
        assert np.array_equal(r["IA"], q["IA"]) and np.array_equal(r["IB"], q["IB"])
        assert np.array_equal(r["U"], q["U"])

    for data in range(2):
        if data == 1:  # different values in the same buffers: reversed rows of A, B scaled and shifted
            At.copy_(torch.from_numpy(np.ascontiguousarray(A[::-1])))
            Bt.copy_(torch.from_numpy((B * 1.5 + 0.25).astype(np.float32)))
        with option("graph", 0):
            ref, n_ref = run()
        for _ in range(3):
            g, n_g = run()
            same(g, ref)
            assert n_g == n_ref
    # a config whose union sizes differ: a new step-4 graph, same answer as eager
    A3, B3 = datagen.generate(2, n=12000)
    At3, Bt3 = torch.from_numpy(A3).cuda(), torch.from_numpy(B3).cuda()
    with option("graph", 0):
        e3 = ctx.prohd_estimate(At3, Bt3, c.k, c.m(12000), return_indices=True)
    g3 = ctx.prohd_estimate(At3, Bt3, c.k, c.m(12000), return_indices=True)
    assert g3["value"] == e3["value"] and np.array_equal(g3["IA"], e3["IA"])


@pytest.mark.parametrize("D", [264, 320])
def test_wide_d_end_to_end(ctx, D):
    """ProHD with k > 0 above D = 256 (Alg. 2 needs only k <= D): the eigen-solver's
    D <= 512 variant, the fp64 DMMA Gram and the SIMT projection; selected sets bit-exact with
    the oracle, the estimate within 1e-4."""
    rng = np.random.default_rng(D)
    n = 6000
    scales = np.geomspace(3.0, 0.1, D)
    A = (rng.standard_normal((n, D)) * scales).astype(np.float32)
    B = (rng.standard_normal((n + 7, D)) * scales + 0.05).astype(np.float32)
    k, m = 8, 30
    g = ctx.prohd_estimate(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), k, m, return_indices=True)
    r = OP.estimate(A, B, k, m)
    assert np.array_equal(g["IA"], r["IA"]) and np.array_equal(g["IB"], r["IB"])
    assert abs(g["value"] - r["value"]) <= 1e-4 * r["value"]
