"""Cyclic Jacobi eigen-solver for a real symmetric matrix, fp64 (own implementation).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Used for Alg. 2 line 2, "Compute the top m principal components": the
principal components of the stacked union are the eigenvectors of its covariance
with the largest eigenvalues. The paper names "randomized or truncated SVD"
 as a way to get them; the oracle instead uses the classical
two-sided Jacobi method (Golub & Van Loan, Alg. 8.5.3 "cyclic Jacobi"), run in a
round-robin ("tournament") ordering so each round applies D/2 disjoint
rotations at once. It is independent of LAPACK (pinned against numpy.linalg.eigh
and closed forms in tests/test_oracle_eigen.py).

Rotation for pair (p, q), Golub & Van Loan Alg. 8.4.1 (sym.schur2):
    tau = (a_qq - a_pp) / (2 a_pq)
    t   = sign(tau) / (|tau| + sqrt(1 + tau^2))      (t = 1 if tau == 0)
    c   = 1 / sqrt(1 + t^2),  s = t c
    A  <- J^T A J,  V <- V J,   J = I except J_pp = J_qq = c, J_pq = s, J_qp = -s.
Sweeps repeat until off(A) = ||A - diag(A)||_F <= tol * ||A||_F.
"""
from __future__ import annotations

import numpy as np


def _tournament(n: int) -> list[tuple[np.ndarray, np.ndarray]]:
    """Round-robin schedule of n (even) players: n-1 rounds of n/2 disjoint pairs."""
    players = list(range(n))
    rounds = []
    for _ in range(n - 1):
        p = np.array(players[: n // 2])
        q = np.array(players[n // 2:][::-1])
        lo, hi = np.minimum(p, q), np.maximum(p, q)
        rounds.append((lo, hi))
        players = [players[0]] + [players[-1]] + players[1:-1]
    return rounds


def jacobi_eigh(C: np.ndarray, tol: float = 1e-15, max_sweeps: int = 60) -> tuple[np.ndarray, np.ndarray]:
    """Eigen-decomposition of symmetric C: returns (w, V), C V = V diag(w).

    Eigenpairs are returned unsorted (in Jacobi's diagonal order); callers sort.
    """
    A = np.array(C, dtype=np.float64, copy=True)
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise ValueError("square matrix required")
    if not np.allclose(A, A.T, rtol=0, atol=1e-12 * (np.abs(A).max() + 1e-300)):
        raise ValueError("matrix not symmetric")
    A = 0.5 * (A + A.T)
    n0 = A.shape[0]
    n = n0 + (n0 % 2)
    if n != n0:  # pad with an isolated zero row/column (already diagonal)
        A = np.pad(A, ((0, 1), (0, 1)))
    V = np.eye(n)
    rounds = _tournament(n) if n > 1 else []
    fro = np.linalg.norm(A)
    if fro == 0.0:
        return np.zeros(n0), np.eye(n0)
    for _ in range(max_sweeps):
        O = A - np.diag(np.diag(A))
        off = np.sqrt(np.sum(O * O))
        if off <= tol * fro:
            break
        for p, q in rounds:
            apq = A[p, q]
            app = A[p, p]
            aqq = A[q, q]
            act = apq != 0.0
            with np.errstate(over="ignore", divide="ignore"):
                tau = np.where(act, (aqq - app) / np.where(act, 2.0 * apq, 1.0), 0.0)
                sgn = np.where(tau >= 0.0, 1.0, -1.0)
                # sqrt(1 + tau^2) as hypot(1, tau): no overflow for |tau| > 1e154 (t -> 0 limit)
                t = np.where(act, sgn / (np.abs(tau) + np.hypot(1.0, tau)), 0.0)
            c = 1.0 / np.sqrt(1.0 + t * t)
            s = t * c
            # A <- A J (columns p, q)
            Ap = A[:, p].copy()
            Aq = A[:, q]
            A[:, p] = c[None, :] * Ap - s[None, :] * Aq
            A[:, q] = s[None, :] * Ap + c[None, :] * Aq
            # A <- J^T A (rows p, q)
            Ap = A[p, :].copy()
            Aq = A[q, :]
            A[p, :] = c[:, None] * Ap - s[:, None] * Aq
            A[q, :] = s[:, None] * Ap + c[:, None] * Aq
            # V <- V J
            Vp = V[:, p].copy()
            Vq = V[:, q]
            V[:, p] = c[None, :] * Vp - s[None, :] * Vq
            V[:, q] = s[None, :] * Vp + c[None, :] * Vq
    w = np.diag(A).copy()
    if n != n0:
        # drop the padded coordinate: its eigenvector is e_n (untouched, apq == 0)
        keep = np.arange(n0)
        w = w[keep]
        V = V[:n0, keep]
    return w, V
