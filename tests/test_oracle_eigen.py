"""Pins for oracle/eigen.py (cyclic Jacobi) — closed forms and LAPACK (numpy.linalg.eigh)."""
import numpy as np
import pytest

from oracle.eigen import jacobi_eigh
from oracle import prohd


def _sorted(w, V):
    o = np.argsort(-w, kind="stable")
    return w[o], V[:, o]


def test_diagonal():
    d = np.array([3.0, -1.0, 7.5, 0.0, 2.0])
    w, V = jacobi_eigh(np.diag(d))
    assert np.allclose(np.sort(w), np.sort(d), atol=0)
    P = np.abs(V)
    assert np.array_equal(np.sort(P, axis=0)[-1], np.ones(5))  # a permutation matrix
    assert np.allclose(np.diag(d) @ V, V * w[None, :], atol=0)


@pytest.mark.parametrize("a,b,c", [(2.0, 1.0, 3.0), (1.0, -4.0, 1.0), (5.0, 1e-8, 5.0), (0.0, 2.0, -3.0)])
def test_2x2_closed_form(a, b, c):
    """lambda = (a+c)/2 +- sqrt(((a-c)/2)^2 + b^2)."""
    w, V = jacobi_eigh(np.array([[a, b], [b, c]]))
    r = np.sqrt(((a - c) / 2) ** 2 + b * b)
    ref = np.array([(a + c) / 2 + r, (a + c) / 2 - r])
    assert np.allclose(np.sort(w)[::-1], ref, rtol=0, atol=1e-14 * max(1, abs(r)))


def test_rank_one():
    rng = np.random.default_rng(0)
    v = rng.standard_normal(9)
    v /= np.linalg.norm(v)
    w, V = _sorted(*jacobi_eigh(4.0 * np.outer(v, v)))
    assert abs(w[0] - 4.0) < 1e-13
    assert np.allclose(np.abs(w[1:]), 0.0, atol=1e-13)
    assert abs(abs(V[:, 0] @ v) - 1.0) < 1e-13


@pytest.mark.parametrize("D", [1, 2, 3, 7, 16, 33, 64])
def test_against_lapack(D):
    rng = np.random.default_rng(D)
    X = rng.standard_normal((4 * D + 5, D)) * (np.arange(1, D + 1) ** -0.5)
    C = X.T @ X / X.shape[0]
    w, V = _sorted(*jacobi_eigh(C))
    wr, Vr = np.linalg.eigh(C)
    wr, Vr = wr[::-1], Vr[:, ::-1]
    scale = max(abs(wr).max(), 1e-300)
    assert np.allclose(w, wr, rtol=0, atol=1e-12 * scale)
    assert np.allclose(V.T @ V, np.eye(D), atol=1e-12)
    assert np.allclose(C @ V, V * w[None, :], atol=1e-12 * scale)
    # gap-scaled angle agreement for separated eigenvalues
    for j in range(D):
        gap = min([abs(wr[j] - wr[i]) for i in range(D) if i != j] + [np.inf])
        if gap > 1e-6 * scale:
            c = V[:, j] @ Vr[:, j]
            s = np.linalg.norm(V[:, j] - c * Vr[:, j])  # sin of the angle
            assert s <= 1e-10 * scale / gap + 1e-12


def test_top_components_sign_and_rank_drop():
    v1 = np.array([0.0, -3.0, 1.0, 0.0])
    v1 /= np.linalg.norm(v1)
    v2 = np.array([1.0, 0.0, 0.0, 1.0]) / np.sqrt(2)
    C = 5 * np.outer(v1, v1) + 2 * np.outer(v2, v2)  # rank 2
    lam, V = prohd.top_components(C, 4)
    assert V.shape[1] == 2  # rank shortfall: only 2 directions
    assert np.allclose(lam, [5, 2])
    assert np.allclose(V[:, 0], -v1)  # largest |coordinate| (index 1) made positive
    assert np.allclose(V[:, 1], v2)  # tie between index 0 and 3 -> lowest index positive
