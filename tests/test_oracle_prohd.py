"""Pins for oracle/prohd.py (Alg. 1-3) and the theorem invariants.

Pins used: hand-worked W3/W4/W5, SPEC examples, naive loops
for centroid/covariance, closed-form special cases (2m >= n reduces to the exact
HD; A = B gives 0), the proven bounds of §III-E for H_U and the subset-full
estimate, and the survey's independent cfg1 recomputation (X2b).
"""
import itertools

import numpy as np
import pytest

import datagen
import oracle
from oracle import prohd


# ------------------------------------------------------------------ O1-O3

def test_centroid_examples():
    assert np.array_equal(prohd.centroid(np.array([[3.0, 4.0]])), [3.0, 4.0])
    assert np.array_equal(prohd.centroid(np.array([[0.0, 0.0], [2.0, 2.0]])), [1.0, 1.0])
    rng = np.random.default_rng(0)
    X = rng.standard_normal((100, 5))
    naive = [sum(X[i, j] for i in range(100)) / 100 for j in range(5)]
    assert np.allclose(prohd.centroid(X), naive, rtol=0, atol=1e-12)


def test_centroid_axis_e1_rule():
    """equal centroids -> u = e1."""
    A = np.array([[1.0, 2.0, 3.0], [3.0, 2.0, 1.0]])
    B = np.array([[2.0, 2.0, 2.0]])
    assert np.array_equal(prohd.centroid_axis(A, B), [1.0, 0.0, 0.0])
    B2 = B + np.array([0.0, 1e-10, 0.0])  # ||d|| < 1e-9 still -> e1
    assert np.array_equal(prohd.centroid_axis(A, B2), [1.0, 0.0, 0.0])
    B3 = B + np.array([0.0, 0.0, -2e-9])
    assert np.allclose(prohd.centroid_axis(A, B3), [0.0, 0.0, -1.0])


def test_covariance_naive_and_shift():
    rng = np.random.default_rng(1)
    A = rng.standard_normal((37, 4))
    B = rng.standard_normal((21, 4)) + 2.0
    Z = np.concatenate([A, B])
    N = Z.shape[0]
    mu = [sum(Z[i, j] for i in range(N)) / N for j in range(4)]
    C = [[sum((Z[i, a] - mu[a]) * (Z[i, b] - mu[b]) for i in range(N)) / N for b in range(4)] for a in range(4)]
    mu_o, C_o = prohd.covariance(A, B)
    assert np.allclose(mu_o, mu, atol=1e-13) and np.allclose(C_o, C, atol=1e-13)
    _, C_s = prohd.covariance(A + 100.0, B + 100.0)
    assert np.allclose(C_s, C_o, atol=1e-10)


# ------------------------------------------------------------------ W3 (full pipeline)

def test_w3_pipeline(golden):
    g = golden["W3"]
    A = np.array(g["A"], np.float32)
    B = A + np.array(g["B_offset"], np.float32)
    d = prohd.directions(A, B, 2)
    assert np.allclose(d["mu"], g["mu"]) and np.allclose(d["C"], g["C"])
    assert np.allclose(d["u0"], g["u0"])
    assert np.allclose(d["U"][:, 1], g["pc1"]) and np.allclose(d["U"][:, 2], g["pc2"])
    for key, k in (("k1_m1", 1), ("k2_m1", 2)):
        e = prohd.estimate(A, B, k, 1)
        assert e["IA"].tolist() == g[key]["IA"] and e["IB"].tolist() == g[key]["IB"]
        assert e["value"] == g[key]["H_hat"]
        assert [e["ab"]["a"], e["ab"]["b"]] == g[key]["ab_witness"]
    mu = np.array(g["mu"])
    assert prohd.delta(A, B, np.array([0.0, 1.0]), center=mu) == g["delta_centered_e2"]
    assert prohd.delta(A, B, np.array([1.0, 0.0]), center=mu) == g["delta_centered_e1"]
    assert prohd.multi_direction_hd(A, B, d["U"]) == g["H_U"]


def test_w4_counterexample(golden):
    g = golden["W4"]
    A = np.array(g["A"], np.float32)
    B = np.array(g["B"], np.float32)
    U = np.array(g["U"])
    e = prohd.estimate(A, B, 0, g["m"], U=U)
    assert e["value"] == g["H_hat_ss"]
    assert oracle.hausdorff(A, B)["value"] == g["H"]
    assert prohd.multi_direction_hd(A, B, U) == g["H_U"]
    assert prohd.delta(A, B, U[:, 0]) == g["delta"]


def test_w5_counterexample(golden):
    g = golden["W5"]
    A = np.array(g["A"], np.float32)
    B = np.array(g["B"], np.float32)
    U = np.array(g["U"])
    e = prohd.estimate(A, B, 1, g["m"], U=U)
    assert e["IA"].tolist() == g["IA"] and e["IB"].tolist() == g["IB"]
    assert abs(e["value"] - g["H_hat_ss"]) < 1e-6  # sqrt(3.25) in fp32-input arithmetic
    assert abs(oracle.hausdorff(A, B)["value"] - g["H"]) < 1e-6
    assert abs(prohd.multi_direction_hd(A, B, U) - g["H_U"]) < 1e-6
    assert abs(prohd.subset_full(A, B, e["IA"], e["IB"]) - g["H_hat_sf"]) < 1e-6


# ------------------------------------------------------------------ selection

def test_select_examples(golden):
    g = golden["SELECT"]
    b, t = prohd.extremes(np.array(g["values"], float), g["m"])
    assert sorted(set(b.tolist()) | set(t.tolist())) == g["union"]
    v = np.arange(10, dtype=float)[::-1].copy()
    b, t = prohd.extremes(v, 2)
    assert len(set(b) | set(t)) == 4
    b, t = prohd.extremes(np.array([1.0, 1.0, 0.0, 1.0]), 2)
    assert b.tolist() == [2, 0] and t.tolist() == [0, 1]  # ties -> lower index


def test_select_properties():
    rng = np.random.default_rng(3)
    X = rng.standard_normal((500, 6))
    U = np.linalg.qr(rng.standard_normal((6, 4)))[0]
    m = 7
    s = prohd.select(X, U, m)
    n = X.shape[0]
    assert min(n, 2 * m) <= s["union"].size <= min(n, 2 * m * U.shape[1])
    assert np.all(np.diff(s["union"]) > 0)
    P = X @ U
    for l in range(U.shape[1]):  # min and max along every direction are kept
        assert np.argmin(P[:, l]) in s["union"] and np.argmax(P[:, l]) in s["union"]
        # the selection is exactly the m extreme values
        b, t = s["lists"][l]
        assert P[b, l].max() <= np.delete(P[:, l], b).min()
        assert P[t, l].min() >= np.delete(P[:, l], t).max()
    s2 = prohd.select(2.0 * X, U, m)  # scale invariance (exact in fp: x2)
    assert np.array_equal(s2["union"], s["union"])
    sall = prohd.select(X[:10], U, 5)  # 2m >= n -> everything
    assert sall["union"].tolist() == list(range(10))


@pytest.mark.parametrize("G", [1, 2, 3, 8])
def test_sharded_selection_equals_single(G):
    """O12 / SURVEY.md §4.2: local top-m per row block + merge == global top-m."""
    rng = np.random.default_rng(G)
    X = rng.standard_normal((997, 5)).astype(np.float32)
    X[500:520] = X[0]  # duplicates -> exact ties across blocks
    U = np.linalg.qr(rng.standard_normal((5, 3)))[0]
    a = prohd.select(X, U, 13)
    b = prohd.sharded_select(X, U, 13, G)
    for (ab, at), (bb, bt) in zip(a["lists"], b["lists"]):
        assert np.array_equal(ab, bb) and np.array_equal(at, bt)
    assert np.array_equal(a["union"], b["union"])


@pytest.mark.parametrize("G", [1, 2, 5])
def test_sharded_exact_equals_single(G):
    rng = np.random.default_rng(10 + G)
    A = rng.standard_normal((301, 4)).astype(np.float32)
    B = rng.standard_normal((150, 4)).astype(np.float32)
    A[200] = A[10]  # tie in the row maxima
    r = oracle.directed_hd(A, B)
    s = prohd.sharded_directed_hd(A, B, G)
    assert (s["dist2"], s["a"], s["b"]) == (r["dist2"], r["a"], r["b"])


# ------------------------------------------------------------------ ProHD special cases

def test_identical_sets_give_zero():
    rng = np.random.default_rng(4)
    A = rng.standard_normal((300, 5)).astype(np.float32)
    e = prohd.estimate(A, A.copy(), 3, 10)
    assert e["value"] == 0.0


def test_full_selection_equals_exact():
    """2m >= n: the subsets are the full sets, so H^ = H exactly."""
    rng = np.random.default_rng(5)
    A = rng.standard_normal((40, 3)).astype(np.float32)
    B = rng.standard_normal((30, 3)).astype(np.float32) + 1
    e = prohd.estimate(A, B, 2, 20)
    h = oracle.hausdorff(A, B)
    assert e["value"] == h["value"]


def test_symmetry_of_estimate():
    rng = np.random.default_rng(6)
    A = rng.standard_normal((400, 4)).astype(np.float32)
    B = (rng.standard_normal((350, 4)) * 1.3 + 0.4).astype(np.float32)
    e1 = prohd.estimate(A, B, 2, 9)
    e2 = prohd.estimate(B, A, 2, 9)
    assert abs(e1["value"] - e2["value"]) <= 1e-12 * e1["value"]


def test_paper_parameters():
    """Alg. 3 line 1: D=4 -> m=2, alpha'=alpha/2."""
    assert prohd.paper_parameters(4, 0.01, 1000) == (2, 10, 5)
    assert prohd.paper_parameters(1, 0.01, 50) == (1, 1, 1)
    assert prohd.paper_parameters(256, 0.01, 100000) == (16, 1000, 62)


# ------------------------------------------------------------------ theorem invariants (§III-E)

@pytest.mark.parametrize("seed", range(8))
def test_bounds_and_monotonicity(seed):
    rng = np.random.default_rng(100 + seed)
    D = int(rng.choice([2, 3, 5, 8]))
    A = rng.standard_normal((int(rng.integers(20, 120)), D)) * rng.uniform(0.5, 2, D)
    B = rng.standard_normal((int(rng.integers(20, 120)), D)) + rng.standard_normal(D)
    H = oracle.hausdorff(A, B)["value"]
    d = prohd.directions(A, B, min(D, 3))
    U = d["U"]
    mu = d["mu"]
    # single direction sandwich for random u, both delta frames
    for _ in range(5):
        u = rng.standard_normal(D)
        u /= np.linalg.norm(u)
        hu = max(prohd.hd_1d(A @ u, B @ u))
        assert hu <= H + 1e-9
        assert H <= hu + 2 * prohd.delta(A, B, u) + 1e-9
        assert H <= hu + 2 * prohd.delta(A, B, u, center=mu) + 1e-9
    # multi-direction bound (Eq. 4) and monotonicity
    prev = -1.0
    prev_delta = np.inf
    for j in range(1, U.shape[1] + 1):
        HU = prohd.multi_direction_hd(A, B, U[:, :j])
        md = min(prohd.delta(A, B, U[:, l], center=mu) for l in range(j))
        assert HU <= H + 1e-9 and H <= HU + 2 * md + 1e-9
        assert HU >= prev - 1e-12 and md <= prev_delta + 1e-12
        prev, prev_delta = HU, md
    # subset-full estimate never exceeds H
    e = prohd.estimate(A.astype(np.float32), B.astype(np.float32), min(D, 3), 3)
    Af, Bf = A.astype(np.float32), B.astype(np.float32)
    assert prohd.subset_full(Af, Bf, e["IA"], e["IB"]) <= oracle.hausdorff(Af, Bf)["value"] + 1e-12


def test_projection_contraction():
    rng = np.random.default_rng(11)
    for a, b in itertools.islice(zip(rng.standard_normal((50, 6)), rng.standard_normal((50, 6))), 50):
        u = rng.standard_normal(6)
        u /= np.linalg.norm(u)
        assert abs(a @ u - b @ u) <= np.linalg.norm(a - b) + 1e-12


# ------------------------------------------------------------------ cfg1 cross-check

def test_cfg1_seed0(golden):
    g = golden["CFG1_SEED0"]
    A, B = datagen.generate(1, seed=0)
    assert datagen.sha256(A).startswith(g["sha256_prefix_A"])
    assert datagen.sha256(B).startswith(g["sha256_prefix_B"])
    h = oracle.hausdorff(A, B)
    assert abs(h["ab"]["dist"] - g["h_ab"]) < 1e-9 and [h["ab"]["a"], h["ab"]["b"]] == g["h_ab_witness"]
    assert abs(h["ba"]["dist"] - g["h_ba"]) < 1e-9 and [h["ba"]["a"], h["ba"]["b"]] == g["h_ba_witness"]
    e = prohd.estimate(A, B, 4, 20)
    assert (e["size_a"], e["size_b"]) == (g["size_a"], g["size_b"])
    assert abs(e["ab"]["dist"] - g["hhat_ab"]) < 1e-9 and [e["ab"]["a"], e["ab"]["b"]] == g["hhat_ab_witness"]
    assert abs(e["ba"]["dist"] - g["hhat_ba"]) < 1e-9 and [e["ba"]["a"], e["ba"]["b"]] == g["hhat_ba_witness"]
    assert np.allclose(e["lam"], g["top_eigenvalues"], atol=1e-4)


# ------------------------------------------------------------------ paper-literal parameters (O11)

def test_estimate_paper_reduces_to_fixed_m():
    """With n small enough that floor(alpha n) and floor(alpha/m_pc n) clamp to the same count,
    the paper-literal estimate is Alg. 3 with that fixed m (O6 with one count)."""
    rng = np.random.default_rng(21)
    A = rng.standard_normal((90, 9)).astype(np.float32)
    B = (rng.standard_normal((80, 9)) + 0.4).astype(np.float32)
    e = prohd.estimate_paper(A, B, 0.01)  # m_pc = 3, counts max(1, 0) = 1 everywhere
    r = prohd.estimate(A, B, 3, 1)
    assert e["k"] == 3 and np.array_equal(e["IA"], r["IA"]) and np.array_equal(e["IB"], r["IB"])
    assert e["value"] == r["value"]


def test_select_counts_per_direction():
    rng = np.random.default_rng(22)
    X = rng.standard_normal((400, 5))
    U = np.linalg.qr(rng.standard_normal((5, 3)))[0]
    s = prohd.select_counts(X, U, [10, 3, 3])
    P = X @ U
    for l, c in enumerate([10, 3, 3]):
        b, t = s["lists"][l]
        assert len(b) == c and len(t) == c
        assert P[b, l].max() <= np.delete(P[:, l], b).min()
        assert P[t, l].min() >= np.delete(P[:, l], t).max()
    assert s["union"].size <= 2 * (10 + 3 + 3)


def test_sampling_draws():
    import datagen
    u = datagen.uniform_sample(1000, 30, seed=1)
    assert u.size == 30 and np.unique(u).size == 30 and u.min() >= 0 and u.max() < 1000
    sy = datagen.systematic_sample(10, 0.34, seed=1)  # stride 2 -> 5 points
    assert sy.size == 5 and np.unique(sy).size == 5
    assert datagen.systematic_sample(1001, 0.01, 3).size == 11  # ceil(n / floor(1/alpha))
    A, B = datagen.random_clouds(50, 40, 4, seed=0)
    assert A.min() >= 0 and A.max() <= 1 and B.min() >= 0.1 and B.max() <= 1.1
