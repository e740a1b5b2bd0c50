"""GPU parity for the exact Hausdorff path (K0 + K6 + K7) through the C ABI.

Bar (BASELINE.json north_star):
  |d2_gpu - d2_ref| <= 1e-5 * (||a||^2 + ||b||^2)
for every checked row minimum (pair = the row and its oracle nearest neighbour)
and for the HD value; the reported witness must be a valid one (its fp64
distance within tolerance of the oracle's value), and the fp64-recomputed
witness column must be the oracle's exact nearest neighbour of that row.
"""
import numpy as np
import pytest
import torch

import datagen
import oracle

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def ctx():
    from paper_2511_18207_b200 import Context
    return Context(0)


def _check_rowmins(A, B, rowmin_gpu, rows=None):
    ref, arg = oracle.row_minima(A, B, rows=rows)
    Ar = A if rows is None else A[rows]
    na = (Ar.astype(np.float64) ** 2).sum(1)
    nb = (B.astype(np.float64) ** 2).sum(1)[arg]
    g = rowmin_gpu if rows is None else rowmin_gpu[rows]
    err = np.abs(g.astype(np.float64) - ref) / (na + nb + 1e-300)
    assert err.max() <= TOL, f"max rel err {err.max():.3e} at row {int(err.argmax())}"
    return err.max()


def _check_directed(A, B, got, ref):
    """got = GPU directed result, ref = oracle directed result."""
    nd = lambda x: float((np.asarray(x, np.float64) ** 2).sum())
    a_star, b_star = ref["a"], ref["b"]
    tol = TOL * (nd(A[a_star]) + nd(B[b_star]))
    assert abs(got["dist2"] - ref["dist2"]) <= tol
    # the GPU's witness row: its exact fp64 row-min equals the reported value,
    # and its column is the oracle's nearest neighbour of that row
    rmin, arg = oracle.row_minima(A, B, rows=np.array([got["a"]]))
    assert got["b"] == int(arg[0])
    assert abs(got["dist2"] - rmin[0]) <= 1e-12 * max(1.0, rmin[0])
    assert abs(got["dist"] - np.sqrt(got["dist2"])) <= 1e-12 * max(1.0, got["dist"])


@pytest.mark.parametrize("shape", [(1, 1, 1), (4, 4, 2), (5, 7, 3), (130, 257, 8), (300, 513, 16),
                                   (129, 255, 20), (1000, 3000, 64), (700, 900, 128), (513, 1100, 256),
                                   (257, 300, 40)])
def test_rowmin_random(ctx, shape):
    nA, nB, D = shape
    rng = np.random.default_rng(nA * 7 + nB * 13 + D)
    A = rng.standard_normal((nA, D)).astype(np.float32)
    B = (rng.standard_normal((nB, D)) * 1.5 + 0.25).astype(np.float32)
    rm = ctx.directed_hd_rowmin(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
    _check_rowmins(A, B, rm)


def test_w3_bit_exact(ctx, golden):
    """W3 values are exact in fp32; the tie rules must reproduce the oracle exactly."""
    g = golden["W3"]
    A = np.array(g["A"], np.float32)
    B = A + np.array(g["B_offset"], np.float32)
    h = ctx.hausdorff(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
    assert h["value"] == g["H"]
    assert [h["ab"]["a"], h["ab"]["b"]] == g["h_ab_witness"]
    assert [h["ba"]["a"], h["ba"]["b"]] == g["h_ba_witness"]


def test_w0_w1(ctx, golden):
    for key in ("W0", "W1"):
        g = golden[key]
        A = torch.tensor(g["A"], dtype=torch.float32).cuda()
        B = torch.tensor(g["B"], dtype=torch.float32).cuda()
        assert ctx.hausdorff(A, B)["value"] == g["H"]
    g = golden["W1"]
    r = ctx.directed_hd(torch.tensor(g["A"], dtype=torch.float32).cuda(),
                        torch.tensor(g["B"], dtype=torch.float32).cuda())
    assert [r["a"], r["b"]] == g["h_ab_witness"] and r["dist"] == g["h_ab"]


def test_cfg1_full(ctx):
    A, B = datagen.generate(1)
    h = ctx.hausdorff(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
    ref = oracle.hausdorff(A, B)
    _check_directed(A, B, h["ab"], ref["ab"])
    _check_directed(B, A, h["ba"], ref["ba"])
    # cfg1's witnesses are robust (top-two row-min gap >> tolerance): identical
    assert (h["ab"]["a"], h["ab"]["b"]) == (ref["ab"]["a"], ref["ab"]["b"])
    assert (h["ba"]["a"], h["ba"]["b"]) == (ref["ba"]["a"], ref["ba"]["b"])
    rm = ctx.directed_hd_rowmin(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
    _check_rowmins(A, B, rm)


def test_host_inputs_match_device_inputs(ctx):
    rng = np.random.default_rng(5)
    A = rng.standard_normal((777, 32)).astype(np.float32)
    B = rng.standard_normal((555, 32)).astype(np.float32)
    hd = ctx.hausdorff(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
    hh = ctx.hausdorff(torch.from_numpy(A), torch.from_numpy(B))  # host pointers -> staged copy
    assert hd == hh


def test_identity_zero_and_symmetry(ctx):
    rng = np.random.default_rng(6)
    A = rng.standard_normal((1500, 64)).astype(np.float32)
    At = torch.from_numpy(A).cuda()
    h = ctx.hausdorff(At, At.clone())
    assert h["value"] == 0.0  # fp64 witness re-evaluation of identical points is exactly 0
    B = rng.standard_normal((900, 64)).astype(np.float32)
    Bt = torch.from_numpy(B).cuda()
    assert ctx.hausdorff(At, Bt)["value"] == ctx.hausdorff(Bt, At)["value"]


def test_determinism(ctx):
    A, B = datagen.generate(2, n=20000)
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    r1 = ctx.hausdorff(At, Bt)
    r2 = ctx.hausdorff(At, Bt)
    assert r1 == r2


def test_errors(ctx):
    from paper_2511_18207_b200 import ProHDError
    A = torch.zeros((4, 3), device="cuda")
    B = torch.zeros((5, 3), device="cuda")
    with pytest.raises(ProHDError) as e:
        ctx.directed_hd(A[:0], B)
    assert e.value.code == 2
    Bn = B.clone()
    Bn[2, 1] = float("nan")
    with pytest.raises(ProHDError) as e:
        ctx.directed_hd(A, Bn)
    assert e.value.code == 3
    Bi = B.clone()
    Bi[0, 0] = float("inf")
    with pytest.raises(ProHDError) as e:
        ctx.hausdorff(A, Bi)
    assert e.value.code == 3


@pytest.mark.parametrize("cfg", [2])
def test_cfg_full_rows(ctx, cfg):
    """cfg2 at full size: every row minimum checked."""
    A, B = datagen.generate(cfg)
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    rm = ctx.directed_hd_rowmin(At, Bt).cpu().numpy()
    _check_rowmins(A, B, rm)
    r = ctx.directed_hd(At, Bt)
    ref_rows = oracle.row_minima(A, B, rows=np.array([r["a"]]))
    assert abs(r["dist2"] - ref_rows[0][0]) <= 1e-12 * ref_rows[0][0]
    # no row's true minimum exceeds the reported value by more than the tolerance
    assert rm.max() <= r["dist2_tc"] + 1e-6


@pytest.mark.parametrize("shape", [(1, 1, 4), (3, 700, 16), (300, 5, 8), (129, 257, 20), (1000, 3000, 64),
                                   (777, 513, 256), (2048, 4099, 128)])
def test_bidirectional_pass_matches_oracle(ctx, shape):
    """f4: hausdorff() runs one fused sweep; its B->A side (column minima) must match the oracle."""
    nA, nB, D = shape
    rng = np.random.default_rng(nA + 3 * nB + 7 * D)
    A = rng.standard_normal((nA, D)).astype(np.float32)
    B = (rng.standard_normal((nB, D)) * 1.3 + 0.2).astype(np.float32)
    h = ctx.hausdorff(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
    ref = oracle.hausdorff(A, B)
    _check_directed(A, B, h["ab"], ref["ab"])
    _check_directed(B, A, h["ba"], ref["ba"])
    d = ctx.directed_hd(torch.from_numpy(B).cuda(), torch.from_numpy(A).cuda())
    tol = 1e-5 * (float((B[d["a"]].astype(np.float64) ** 2).sum()) + float((A[d["b"]].astype(np.float64) ** 2).sum()))
    assert abs(h["ba"]["dist2"] - d["dist2"]) <= tol


@pytest.mark.parametrize("split3", [0, 1])
@pytest.mark.parametrize("kind", ["positive", "heavy", "offset"])
def test_split_product_error_bound(ctx, kind, split3):
    """K6 forms a.b as hi.hi + hi.lo + lo.hi on K0's split operands (fp16 of the power-of-two-scaled
    coordinates by default, RN-TF32 fp32 with option k6_split3): 11 + 11 significant bits, error per
    product <= 3 2^-22 |a_i||b_i|, plus the tensor core's fp32 accumulation (<= ~2^-23 |acc| per
    MMA, 3 D / 16 or 3 D / 8 MMAs) -- on the centred operands (c = fp64 mean of the first <= 4096
    rows of B). Inputs chosen so the rounding errors tend to align: all-positive
    data with every mantissa bit in play, heavy tails, and a large common offset."""
    from paper_2511_18207_b200 import option
    rng = np.random.default_rng({"positive": 1, "heavy": 2, "offset": 3}[kind])
    nA, nB, D = 1536, 2048, 256
    if kind == "positive":
        A = (1.0 + rng.random((nA, D)) * 0.999).astype(np.float32)
        B = (1.0 + rng.random((nB, D)) * 0.999).astype(np.float32)
    elif kind == "heavy":
        A = (rng.standard_t(2, (nA, D)) * 3).astype(np.float32)
        B = (rng.standard_t(2, (nB, D)) * 3 + 0.5).astype(np.float32)
    else:
        A = (rng.standard_normal((nA, D)) + 1000.0).astype(np.float32)
        B = (rng.standard_normal((nB, D)) + 1000.25).astype(np.float32)
    with option("k6_split3", split3):
        rm = ctx.directed_hd_rowmin(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
    ref, arg = oracle.row_minima(A, B)
    c = B[: min(nB, 4096)].astype(np.float64).mean(0)
    na = ((A.astype(np.float64) - c) ** 2).sum(1)
    nb = ((B.astype(np.float64)[arg] - c) ** 2).sum(1)
    err = np.abs(rm.astype(np.float64) - ref)
    nmma = 3 * D / (8 if split3 else 16)
    bound = (3 * 2.0 ** -22 + nmma / 2 * 2.0 ** -23 + 4 * 2.0 ** -24) * (na + nb)
    assert np.all(err <= bound), f"max err / bound {np.max(err / bound):.3f}"
    raw = (A.astype(np.float64) ** 2).sum(1) + (B.astype(np.float64)[arg] ** 2).sum(1)
    assert np.all(err <= TOL * raw)
    print(f"{kind} split3={split3}: max err / (centred bound) = {np.max(err / bound):.3e}")


def _fp16_split_rel_err(x):
    """CPU emulation of K0's default split for the product x.x (one power-of-two scale putting
    max |x| into (2^13, 2^14], hi = fp16(s x), lo = fp16(s x - hi), exact products, lo.lo dropped)."""
    m = float(np.max(np.abs(x)))
    s = 2.0 ** (14 - np.frexp(m)[1])
    y = x.astype(np.float64) * s
    hi = y.astype(np.float16).astype(np.float64)
    lo = (y - hi).astype(np.float16).astype(np.float64)
    return (hi * hi + 2 * hi * lo - y * y) / (y * y)


def test_split_worst_case_mantissas(ctx):
    """Adversarial split-precision case: rows of D = 256 equal coordinates
    x, so every product's rounding error and every accumulator truncation has the same sign and
    the d^2 error of the pair (x.1, x.1) is 2 D err(x.x) x^2 + the accumulation error, against the
    Q17 budget 1e-5 (2 D x^2). Mantissas: the 16 worst of the earlier TF32 + bf16-pair split (the
    worst case 1.0048771f was 1.22e-5 of the product alone), the 16 worst of an exhaustive
    emulation of the current fp16 split, and 32 random ones, at three binades and both signs.
    B = {x.1, -x.1} per x so the centre K0 subtracts is exactly 0. Checked for the default split and
    for the literal 3xTF32 option."""
    from paper_2511_18207_b200 import option
    m = np.arange(1 << 23, dtype=np.uint32)
    xs = (m | np.uint32(127 << 23)).view(np.float32)
    e16 = _fp16_split_rel_err(xs)
    assert np.abs(e16).max() <= 3 * 2.0 ** -22
    old = np.array([1.0048771, 1.0043917, 1.0043879, 1.0112314, 1.0200167, 1.0200129, 1.0268564], np.float32)
    rng = np.random.default_rng(0)
    vals = np.concatenate([old, xs[np.argsort(-np.abs(e16))[:16]], xs[rng.integers(0, 1 << 23, 32)]])
    vals = np.concatenate([vals * np.float32(s) for s in (0.125, 1.0, 32.0)] +
                          [-vals * np.float32(4.0)]).astype(np.float32)
    D = 256
    worst = {}
    for split3 in (0, 1):
        errs = []
        with option("k6_split3", split3):
            for x in vals:  # one x per call: the self pair is the row's only near neighbour
                A = np.full((1, D), x, np.float32)
                B = np.concatenate([A, -A])
                rm = ctx.directed_hd_rowmin(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
                errs.append(float(rm[0]) / (2 * D * float(x) ** 2))  # exact d2 = 0
        worst[split3] = max(errs)
        assert worst[split3] <= TOL, (split3, worst[split3], vals[int(np.argmax(errs))])
    print(f"worst-case mantissas: max |d2 err| / Q17 budget: default {worst[0] / TOL:.3f}, "
          f"3xTF32 {worst[1] / TOL:.3f}")


@pytest.mark.parametrize("shape", [(333, 1000, 300), (200, 700, 513), (129, 300, 1000)])
def test_rowmin_wide(ctx, shape):
    """D > 256 (several passes of the K-chunk loop, zero-padded ragged last chunk)."""
    nA, nB, D = shape
    rng = np.random.default_rng(D)
    A = rng.standard_normal((nA, D)).astype(np.float32)
    B = (rng.standard_normal((nB, D)) + 0.1).astype(np.float32)
    rm = ctx.directed_hd_rowmin(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
    _check_rowmins(A, B, rm)


@pytest.fixture
def split3():
    """option k6_split3 = 1: the north star's literal 3xTF32 form (three TF32 MMAs on fp32 hi/lo)."""
    from paper_2511_18207_b200 import option
    with option("k6_split3", 1):
        yield


@pytest.mark.parametrize("shape", [(300, 513, 16), (1000, 3000, 64), (513, 1100, 256), (2000, 2500, 128)])
def test_rowmin_literal_3xtf32(ctx, split3, shape):
    nA, nB, D = shape
    rng = np.random.default_rng(nA + D)
    A = rng.standard_normal((nA, D)).astype(np.float32)
    B = (rng.standard_normal((nB, D)) * 1.5 + 0.25).astype(np.float32)
    rm = ctx.directed_hd_rowmin(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
    _check_rowmins(A, B, rm)
    h = ctx.hausdorff(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
    ref = oracle.hausdorff(A, B)
    _check_directed(A, B, h["ab"], ref["ab"])
    _check_directed(B, A, h["ba"], ref["ba"])


@pytest.mark.parametrize("D", [16, 64, 256])
def test_wide_dynamic_range_per_row_scales(ctx, D):
    """K0's per-row scale mode (internal.cuh prep_mode_perrow): a tight cluster of tiny points
    (coordinates ~1e-6) next to far outliers (coordinates 1e4). One fp16 scale per set would leave the
    cluster's coordinates in the fp16 subnormal range (floor 2^-38 x 1e4 per coordinate, ~1e-3 of
    their size); per-row scales keep every row at the top of the range. Both directions of the
    fused sweep and the directed kernel are checked per row against the oracle (Q17); the HD values
    and witnesses too (the outliers sit 0.5 apart per coordinate, so they carry H: with exactly
    coincident outliers H would be a cluster distance ~1e-5, below the fp32 accumulation error
    that Q17 allows on the outliers' own row minima, ~1e-7 of their norms)."""
    rng = np.random.default_rng(D + 5)
    A = (rng.standard_normal((700, D)) * 1e-6).astype(np.float32)
    B = (rng.standard_normal((900, D)) * 1e-6 + 2e-7).astype(np.float32)
    A[3], A[4] = 1e4, -1e4  # symmetric outliers: the centres K0 subtracts stay ~0, so the cluster's
    B[5], B[600] = -1e4 - 0.5, 1e4 + 0.5  # centred norms are its raw norms (the Q17 scale)
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    rm = ctx.directed_hd_rowmin(At, Bt).cpu().numpy()
    _check_rowmins(A, B, rm)
    h, r1, c1 = ctx.hausdorff_minima(At, Bt)
    _check_rowmins(A, B, r1.cpu().numpy())
    _check_rowmins(B, A, c1.cpu().numpy())
    ref = oracle.hausdorff(A, B)
    _check_directed(A, B, h["ab"], ref["ab"])
    _check_directed(B, A, h["ba"], ref["ba"])


def test_graph_replay_exact(ctx):
    """directed_hd / hausdorff replay a cached CUDA graph of their whole enqueue on device inputs:
    repeated calls and new values in the same buffers return exactly the eager result (option
    graph = 0)."""
    from paper_2511_18207_b200 import option
    rng = np.random.default_rng(31)
    A = rng.standard_normal((3001, 64)).astype(np.float32)
    B = (rng.standard_normal((2500, 64)) + 0.3).astype(np.float32)
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    for data in range(2):
        if data == 1:
            At.copy_(torch.from_numpy((A * 2.0 - 1.0).astype(np.float32)))
            Bt.copy_(torch.from_numpy(np.ascontiguousarray(B[::-1])))
        with option("graph", 0):
            d0, h0 = ctx.directed_hd(At, Bt), ctx.hausdorff(At, Bt)
        for _ in range(3):
            assert ctx.directed_hd(At, Bt) == d0
            assert ctx.hausdorff(At, Bt) == h0


@pytest.mark.parametrize("shape", [(1, 1, 128), (5, 300, 130), (257, 513, 256), (700, 2000, 128),
                                   (513, 1100, 256), (129, 40000, 256), (20000, 3001, 200)])
def test_rowmin_cta_pair(ctx, shape):
    """The CTA-pair K6 (option k6_variant = 2: M=256 cta_group::2 MMAs, double-buffered 256-column
    accumulators, B split across the pair): per-row Q17 against the oracle on ragged shapes (partial
    256-row blocks, a single row, column-split units merged by atomicMin, feature counts off the
    32-feature stage), the HD witness, and the per-row scale mode."""
    from paper_2511_18207_b200 import option
    nA, nB, D = shape
    rng = np.random.default_rng(nA * 3 + nB + D)
    A = rng.standard_normal((nA, D)).astype(np.float32)
    B = (rng.standard_normal((nB, D)) * 1.5 + 0.25).astype(np.float32)
    rows = None if nA * nB <= 4_000_000 else np.unique(rng.integers(0, nA, 400))
    with option("k6_variant", 2):
        At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        rm = ctx.directed_hd_rowmin(At, Bt).cpu().numpy()
        got = ctx.directed_hd(At, Bt)
    _check_rowmins(A, B, rm, rows=rows)
    if rows is None:
        ref = oracle.hausdorff(A, B)["ab"]
        _check_directed(A, B, got, ref)
    with option("k6_variant", 3):
        rm3 = ctx.directed_hd_rowmin(At, Bt).cpu().numpy()
    # same arithmetic per pair (three fp16 MMAs, fp32 accumulation in the same K order)
    assert np.array_equal(rm, rm3)


def test_rowmin_cta_pair_per_row_scales(ctx):
    from paper_2511_18207_b200 import option
    rng = np.random.default_rng(77)
    A = (rng.standard_normal((700, 256)) * 1e-6).astype(np.float32)
    B = (rng.standard_normal((900, 256)) * 1e-6 + 2e-7).astype(np.float32)
    A[3], A[4] = 1e4, -1e4
    B[5], B[600] = -1e4 - 0.5, 1e4 + 0.5
    with option("k6_variant", 2):
        rm = ctx.directed_hd_rowmin(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
    _check_rowmins(A, B, rm)


@pytest.mark.parametrize("shape", [(1, 1, 128), (5, 300, 130), (257, 513, 256), (777, 513, 256),
                                   (2048, 4099, 128), (129, 40000, 256), (20000, 3001, 200)])
def test_bidirectional_cta_pair(ctx, shape):
    """The fused bidirectional sweep on the CTA-pair K6 (option k6_bidir_2a = 2): hausdorff() against
    the oracle in both directions on ragged shapes (partial 256-row blocks, rows past nA excluded from
    the column minima, column-split units), and row / column minima bit-identical to the single-block
    sweep (same three fp16 MMAs per accumulator element in the same K order; min is order-free)."""
    from paper_2511_18207_b200 import option
    nA, nB, D = shape
    rng = np.random.default_rng(nA + 5 * nB + 11 * D)
    A = rng.standard_normal((nA, D)).astype(np.float32)
    B = (rng.standard_normal((nB, D)) * 1.3 + 0.2).astype(np.float32)
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    with option("k6_bidir_2a", 2):
        h, rm, cm = ctx.hausdorff_minima(At, Bt)
    with option("k6_bidir_2a", 0):
        h1, rm1, cm1 = ctx.hausdorff_minima(At, Bt)
    assert torch.equal(rm, rm1) and torch.equal(cm, cm1)
    assert h == h1
    if nA * nB <= 4_000_000:
        ref = oracle.hausdorff(A, B)
        _check_directed(A, B, h["ab"], ref["ab"])
        _check_directed(B, A, h["ba"], ref["ba"])
    else:
        _check_rowmins(A, B, rm.cpu().numpy(), rows=np.unique(rng.integers(0, nA, 300)))
        _check_rowmins(B, A, cm.cpu().numpy(), rows=np.unique(rng.integers(0, nB, 300)))
