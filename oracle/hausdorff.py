"""Exact Hausdorff distance, Eq. (1), in fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

    h(A,B) = max_{a in A} min_{b in B} ||a - b||_2
    H(A,B) = max{ h(A,B), h(B,A) }

Tie rules: the nearest neighbour of a row is
the LOWEST column index among exactly-equal fp64 distances; the directed maximum
is the LOWEST row index among exactly-equal row minima; the undirected witness is
the A->B one when h(A,B) == h(B,A).

Evaluation: the fp32 inputs are upcast exactly to fp64. Per block, squared
distances are screened in the expanded form ||a||^2 + ||b||^2 - 2 a.b (one BLAS
GEMM); every column within `SCREEN_TOL * (||a||^2 + max||b||^2)` of the block's
running row minimum is re-evaluated in the direct form sum_k (a_k - b_k)^2, and
only direct-form values decide the minimum. The expanded form's fp64 error is
~ (D+2) * 2^-52 * (||a||^2 + ||b||^2) << SCREEN_TOL, so no true minimiser is
screened out. Pins: tests/test_oracle_hausdorff.py (hand examples W0/W1/W3,
scipy's directed_hausdorff, naive brute force, invariants).
"""
from __future__ import annotations

import numpy as np

SCREEN_TOL = 1e-12


def _direct_d2(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    diff = a - b
    return np.einsum("ij,ij->i", diff, diff)


def row_minima(A: np.ndarray, B: np.ndarray, rows: np.ndarray | None = None,
               row_block: int = 256, col_block: int = 32768) -> tuple[np.ndarray, np.ndarray]:
    """For each selected row a_i of A: (min_j ||a_i - b_j||^2, lowest argmin j), fp64.

    `rows` selects a subset of A's rows (default: all). Returns arrays aligned with
    `rows`.
    """
    A64 = np.asarray(A, dtype=np.float64)
    B64 = np.asarray(B, dtype=np.float64)
    if A64.ndim != 2 or B64.ndim != 2 or A64.shape[1] != B64.shape[1]:
        raise ValueError("A and B must be 2-D with equal D")
    if rows is None:
        rows = np.arange(A64.shape[0])
    rows = np.asarray(rows, dtype=np.int64)
    nb = np.einsum("ij,ij->i", B64, B64)
    nbmax = float(nb.max()) if nb.size else 0.0
    best = np.full(rows.size, np.inf)
    arg = np.full(rows.size, -1, dtype=np.int64)
    for r0 in range(0, rows.size, row_block):
        ridx = rows[r0:r0 + row_block]
        Ab = A64[ridx]
        na = np.einsum("ij,ij->i", Ab, Ab)
        tol = SCREEN_TOL * (na + nbmax) + 1e-300
        bbest = best[r0:r0 + row_block]
        barg = arg[r0:r0 + row_block]
        for c0 in range(0, B64.shape[0], col_block):
            Bc = B64[c0:c0 + col_block]
            E = na[:, None] + nb[None, c0:c0 + col_block] - 2.0 * (Ab @ Bc.T)
            thr = np.minimum(E.min(axis=1), bbest) + tol
            ri, cj = np.nonzero(E <= thr[:, None])
            d2 = _direct_d2(Ab[ri], Bc[cj])
            gj = cj + c0
            # per row: smallest d2, then lowest column (lexsort: last key primary)
            order = np.lexsort((gj, d2, ri))
            ri, d2, gj = ri[order], d2[order], gj[order]
            first = np.ones(ri.size, dtype=bool)
            first[1:] = ri[1:] != ri[:-1]
            ri, d2, gj = ri[first], d2[first], gj[first]
            better = d2 < bbest[ri]  # strict: earlier (lower) columns win exact ties
            bbest[ri[better]] = d2[better]
            barg[ri[better]] = gj[better]
    return best, arg


def directed_hd(A: np.ndarray, B: np.ndarray, return_rows: bool = False, **kw) -> dict:
    """h(A,B) with witness (a*, b*): Eq. (1).

    Returns {"dist", "dist2", "a", "b"} (+ "rowmin2", "argmin" if return_rows).
    """
    rmin, arg = row_minima(A, B, **kw)
    i = int(np.argmax(rmin))  # first (lowest) index among equal maxima
    out = {"dist": float(np.sqrt(rmin[i])), "dist2": float(rmin[i]), "a": i, "b": int(arg[i])}
    if return_rows:
        out["rowmin2"] = rmin
        out["argmin"] = arg
    return out


def hausdorff(A: np.ndarray, B: np.ndarray, **kw) -> dict:
    """H(A,B) = max(h(A,B), h(B,A)), Eq. (1); A->B witness on equality."""
    ab = directed_hd(A, B, **kw)
    ba = directed_hd(B, A, **kw)
    val = ab if ab["dist2"] >= ba["dist2"] else ba
    return {"value": val["dist"], "ab": ab, "ba": ba}
