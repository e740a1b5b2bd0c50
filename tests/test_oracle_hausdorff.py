"""Pins for oracle/hausdorff.py (exact HD, Eq. (1)).

Each pin is independent of the oracle's own arithmetic: hand-worked values,
scipy's directed_hausdorff (a different algorithm), a naive double loop in
plain Python, and the invariants the definition implies (identity, symmetry,
rigid-motion invariance).
"""
import math

import numpy as np
import pytest
from scipy.spatial.distance import directed_hausdorff

import oracle


def _naive(A, B):
    """max_i min_j sqrt(sum_k (a_ik - b_jk)^2), lowest-index ties, pure Python."""
    best, bi, bj = -1.0, -1, -1
    for i, a in enumerate(A.tolist()):
        m, mj = math.inf, -1
        for j, b in enumerate(B.tolist()):
            d = sum((x - y) ** 2 for x, y in zip(a, b))
            if d < m:
                m, mj = d, j
        if m > best:
            best, bi, bj = m, i, mj
    return math.sqrt(best), bi, bj


def test_w0(golden):
    g = golden["W0"]
    A = np.array(g["A"], np.float32)
    B = np.array(g["B"], np.float32)
    assert oracle.hausdorff(A, B)["value"] == g["H"]


def test_w1_directed_and_ties(golden):
    g = golden["W1"]
    A = np.array(g["A"], np.float32)
    B = np.array(g["B"], np.float32)
    ab = oracle.directed_hd(A, B)
    ba = oracle.directed_hd(B, A)
    assert ab["dist"] == g["h_ab"] and [ab["a"], ab["b"]] == g["h_ab_witness"]
    assert ba["dist"] == g["h_ba"] and [ba["a"], ba["b"]] == g["h_ba_witness"]
    assert oracle.hausdorff(A, B)["value"] == g["H"]


def test_w3_witnesses(golden):
    g = golden["W3"]
    A = np.array(g["A"], np.float32)
    B = A + np.array(g["B_offset"], np.float32)
    h = oracle.hausdorff(A, B)
    assert h["value"] == g["H"]
    assert [h["ab"]["a"], h["ab"]["b"]] == g["h_ab_witness"]
    assert [h["ba"]["a"], h["ba"]["b"]] == g["h_ba_witness"]


@pytest.mark.parametrize("seed", range(6))
def test_against_scipy(seed):
    rng = np.random.default_rng(seed)
    n, m, D = rng.integers(1, 300), rng.integers(1, 300), int(rng.choice([1, 2, 4, 8, 16, 20]))
    A = rng.standard_normal((n, D)).astype(np.float32)
    B = (rng.standard_normal((m, D)) + 0.3).astype(np.float32)
    r = oracle.directed_hd(A, B)
    ref = directed_hausdorff(A.astype(np.float64), B.astype(np.float64))[0]
    assert abs(r["dist"] - ref) <= 1e-12 * max(1.0, ref)


@pytest.mark.parametrize("seed", range(25))
def test_against_naive_bruteforce(seed):
    rng = np.random.default_rng(1000 + seed)
    n, m = int(rng.integers(1, 60)), int(rng.integers(1, 60))
    D = int(rng.choice([1, 2, 3, 5, 8]))
    A = rng.standard_normal((n, D)).astype(np.float32)
    B = rng.standard_normal((m, D)).astype(np.float32)
    if seed % 3 == 0:  # force exact duplicates -> tie rules matter
        B[: min(m, n) // 2] = A[: min(m, n) // 2]
        A = np.concatenate([A, A[:2]])
    d, i, j = _naive(A.astype(np.float64), B.astype(np.float64))
    r = oracle.directed_hd(A, B)
    assert abs(r["dist"] - d) <= 1e-12 * max(1.0, d)
    assert (r["a"], r["b"]) == (i, j)


def test_identity_and_symmetry():
    rng = np.random.default_rng(7)
    A = rng.standard_normal((150, 12)).astype(np.float32)
    B = rng.standard_normal((90, 12)).astype(np.float32)
    assert oracle.hausdorff(A, A)["value"] == 0.0
    assert oracle.hausdorff(A, B)["value"] == oracle.hausdorff(B, A)["value"]


def test_rigid_motion_invariance():
    rng = np.random.default_rng(8)
    A = rng.standard_normal((120, 6))
    B = rng.standard_normal((100, 6)) + 0.5
    q, r = np.linalg.qr(rng.standard_normal((6, 6)))
    t = rng.standard_normal(6) * 10
    H0 = oracle.hausdorff(A, B)["value"]
    H1 = oracle.hausdorff(A @ q + t, B @ q + t)["value"]
    assert abs(H0 - H1) <= 1e-9 * H0


def test_column_blocking_and_ties():
    """Blocked scan over B columns keeps the lowest index among exact ties."""
    rng = np.random.default_rng(9)
    B = rng.standard_normal((50, 4)).astype(np.float32)
    B = np.concatenate([B, B, B])  # each point appears 3x
    A = B[:10] + np.float32(0.0)
    rmin, arg = oracle.row_minima(A, B, col_block=7)
    assert np.all(rmin == 0.0)
    assert np.array_equal(arg, np.arange(10))


def test_row_subset():
    rng = np.random.default_rng(10)
    A = rng.standard_normal((80, 5))
    B = rng.standard_normal((70, 5))
    full, farg = oracle.row_minima(A, B)
    rows = np.array([3, 17, 79])
    sub, sarg = oracle.row_minima(A, B, rows=rows)
    assert np.array_equal(sub, full[rows]) and np.array_equal(sarg, farg[rows])
