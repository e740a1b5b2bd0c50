"""ProHD (Alg. 1-3 of arxiv 2511.18207) step by step, fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Notation follows BASELINE.json / SURVEY.md §0: `k` = number of principal
directions (the paper's m = floor(sqrt(D))), `m` = points kept per
(set, direction, tail) (the paper's k_X = max{1, floor(alpha n_X)}), and the
direction matrix U = [u0 u1 ... uk] (D x (k+1)); u0 is the centroid axis.

Steps:
  O1  centroids mu_A, mu_B                                   Alg.1 l.1
  O2  u0 = (mu_B - mu_A)/||.||, e1 if ||.|| < 1e-9           Alg.1 l.2
  O3  C = (1/(nA+nB)) sum_{p in A u B} (p-mu)(p-mu)^T        Alg.2 l.1-2
  O4  top-k eigenvectors of C (cyclic Jacobi), sorted by (-lambda, position),
      sign: largest-|coordinate| entry positive (lowest index on ties);
      directions with lambda <= D 2^-52 lambda_1 dropped
  O5  U = [u0, v1..vk]
  O6  per set X and direction l: pi = X u_l (fp64); bottom = first m by
      (pi asc, idx asc), top = first m by (pi desc, idx asc); all of X if 2m >= n_X
                                                             Alg.1 l.5-9, Alg.2 l.5-11
  O7  I_X = sorted unique union over l and tails
  O8  A_sel = A[I_A], B_sel = B[I_B]
  O9  h^(A_sel,B_sel), h^(B_sel,A_sel), H^ = max
  O10 invariant-only extras: H_U, delta(u) (Eq. 2),
      subset-full estimate H^_sf
  O11 paper-literal parameters (m_pc = floor(sqrt D), alpha / alpha/m_pc)
  O12 sharded simulation: per-block local top/bottom-m, merge -> equals O6
"""
from __future__ import annotations

import numpy as np

from .eigen import jacobi_eigh
from .hausdorff import directed_hd, row_minima

CENTROID_EPS = 1e-9  # P:198 "If ||u|| < 10^-9, set u = e1"
_BLOCK = 8192


# ---------------------------------------------------------------- O1 / O3

def centroid(X: np.ndarray) -> np.ndarray:
    """O1: (1/n) sum_i X_i in fp64 (Alg. 1 line 1).

    Blocked: each block of rows is summed in fp64, then the block sums are added
    pairwise (numpy's pairwise reduction along a contiguous axis).
    """
    X = np.asarray(X)
    parts = [np.asarray(X[i:i + _BLOCK], dtype=np.float64).sum(axis=0)
             for i in range(0, X.shape[0], _BLOCK)]
    S = np.ascontiguousarray(np.stack(parts).T).sum(axis=1)
    return S / X.shape[0]


def covariance(A: np.ndarray, B: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """O3: mu of the stacked union Z~=[A;B] and C = (1/N) sum (p-mu)(p-mu)^T (two-pass).

    P:231 "Stack points Z~ = [X;Y]", "Compute the top m principal
    components" — the components are eigenvectors of this covariance
    (centred, 1/N normalisation).
    """
    nA, nB = A.shape[0], B.shape[0]
    mu = (nA * centroid(A) + nB * centroid(B)) / (nA + nB)
    D = A.shape[1]
    C = np.zeros((D, D))
    for X in (A, B):
        for i in range(0, X.shape[0], _BLOCK):
            Y = np.asarray(X[i:i + _BLOCK], dtype=np.float64) - mu[None, :]
            C += Y.T @ Y
    C /= (nA + nB)
    return mu, 0.5 * (C + C.T)


# ---------------------------------------------------------------- O2 / O4 / O5

def centroid_axis(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """O2: u = ybar - xbar normalised; e1 if ||u|| < 1e-9 (Alg. 1 line 2)."""
    d = centroid(B) - centroid(A)
    nrm = np.linalg.norm(d)
    if nrm < CENTROID_EPS:
        u = np.zeros_like(d)
        u[0] = 1.0
        return u
    return d / nrm


def fix_sign(v: np.ndarray) -> np.ndarray:
    """Largest-|coordinate| entry positive; lowest index on ties."""
    j = int(np.argmax(np.abs(v)))
    return -v if v[j] < 0 else v


def top_components(C: np.ndarray, k: int) -> tuple[np.ndarray, np.ndarray]:
    """O4: top-k eigenpairs of C: (lambda desc, V D x k'), k' <= k after rank drop."""
    w, V = jacobi_eigh(C)
    order = np.lexsort((np.arange(w.size), -w))  # (-lambda asc, position asc)
    w, V = w[order], V[:, order]
    D = C.shape[0]
    lam1 = w[0] if w.size else 0.0
    keep = []
    for j in range(min(k, w.size)):
        if w[j] <= D * 2.0 ** -52 * lam1 or lam1 <= 0.0:
            break
        keep.append(j)
    V = V[:, keep]
    out = np.empty_like(V)
    for j in range(V.shape[1]):
        v = V[:, j] / np.linalg.norm(V[:, j])
        out[:, j] = fix_sign(v)
    return w[keep], out


def directions(A: np.ndarray, B: np.ndarray, k: int) -> dict:
    """O1-O5: U = [u0, v1..vk] plus the intermediate quantities."""
    u0 = centroid_axis(A, B)
    mu, C = covariance(A, B)
    lam, V = top_components(C, k) if k > 0 else (np.zeros(0), np.zeros((A.shape[1], 0)))
    U = np.concatenate([u0[:, None], V], axis=1)
    return {"U": U, "u0": u0, "mu": mu, "C": C, "lam": lam,
            "mu_A": centroid(A), "mu_B": centroid(B)}


# ---------------------------------------------------------------- O6 / O7

def project(X: np.ndarray, U: np.ndarray) -> np.ndarray:
    """pi_u(p) = p^T u for every row and direction, fp64: n x (k+1)."""
    return np.asarray(X, dtype=np.float64) @ np.asarray(U, dtype=np.float64)


def extremes(pi: np.ndarray, m: int) -> tuple[np.ndarray, np.ndarray]:
    """O6 for one direction: (bottom, top) index lists of length min(m, n).

    bottom = first m of argsort(pi) (stable: ties -> lower index); top = first m of
    argsort(-pi) (stable). Alg. 1 lines 6-9 ("argsort ... increasing"; keep the
    smallest k_X and largest k_X).
    """
    n = pi.size
    if m < 1:
        raise ValueError("m must be >= 1")
    mm = min(m, n)
    bottom = np.argsort(pi, kind="stable")[:mm]
    top = np.argsort(-pi, kind="stable")[:mm]
    return bottom, top


def select(X: np.ndarray, U: np.ndarray, m: int) -> dict:
    """O6+O7 for one set: per-direction lists and the sorted unique union I_X.

    If 2m >= n_X every point is selected (SURVEY.md §8(b) semantics).
    """
    n = X.shape[0]
    P = project(X, U)
    lists = []
    for l in range(U.shape[1]):
        lists.append(extremes(P[:, l], m))
    if 2 * m >= n:
        union = np.arange(n, dtype=np.int64)
    else:
        union = np.unique(np.concatenate([np.concatenate(t) for t in lists])).astype(np.int64)
    return {"lists": lists, "union": union, "proj": P}


# ---------------------------------------------------------------- O8 / O9

def subset_hd(A: np.ndarray, B: np.ndarray, IA: np.ndarray, IB: np.ndarray) -> dict:
    """O8+O9: H^ = max(h(A_sel,B_sel), h(B_sel,A_sel)), witnesses as ORIGINAL indices."""
    As, Bs = A[IA], B[IB]
    ab = directed_hd(As, Bs)
    ba = directed_hd(Bs, As)
    ab = {**ab, "a": int(IA[ab["a"]]), "b": int(IB[ab["b"]])}
    ba = {**ba, "a": int(IB[ba["a"]]), "b": int(IA[ba["b"]])}  # a in B, b in A
    value = ab["dist"] if ab["dist2"] >= ba["dist2"] else ba["dist"]
    return {"value": value, "ab": ab, "ba": ba}


def estimate(A: np.ndarray, B: np.ndarray, k: int, m: int, U: np.ndarray | None = None) -> dict:
    """Alg. 3 ProjHausdorff in the north-star parameterisation (k PCs, m per tail).

    If `U` is given (D x (k'+1), column 0 the centroid axis) it is used instead of
    O1-O5 ("direction injection").
    """
    info: dict = {}
    if U is None:
        info = directions(A, B, k)
        U = info["U"]
    sA = select(A, U, m)
    sB = select(B, U, m)
    hd = subset_hd(A, B, sA["union"], sB["union"])
    return {"value": hd["value"], "ab": hd["ab"], "ba": hd["ba"],
            "IA": sA["union"], "IB": sB["union"], "size_a": int(sA["union"].size),
            "size_b": int(sB["union"].size), "U": U, "n_dirs": int(U.shape[1]),
            "lists_A": sA["lists"], "lists_B": sB["lists"], **{k_: v for k_, v in info.items() if k_ != "U"}}


# ---------------------------------------------------------------- O10 extras

def hd_1d(pa: np.ndarray, pb: np.ndarray) -> tuple[float, float]:
    """(h_u(A,B), h_u(B,A)) for projected scalars, by sorted merge."""
    def directed(x, y):
        ys = np.sort(y)
        pos = np.searchsorted(ys, x)
        lo = ys[np.clip(pos - 1, 0, ys.size - 1)]
        hi = ys[np.clip(pos, 0, ys.size - 1)]
        return float(np.max(np.minimum(np.abs(x - lo), np.abs(x - hi))))
    return directed(pa, pb), directed(pb, pa)


def multi_direction_hd(A: np.ndarray, B: np.ndarray, U: np.ndarray) -> float:
    """H_U(A,B) = max_{u in U} H_u(A,B)."""
    PA, PB = project(A, U), project(B, U)
    return max(max(hd_1d(PA[:, l], PB[:, l])) for l in range(U.shape[1]))


def delta(A: np.ndarray, B: np.ndarray, u: np.ndarray, center: np.ndarray | None = None) -> float:
    """delta(u) = max_{p in A u B} ||p - pi_u(p) u|| (Eq. 2).

    `center=None` is the literal (through-the-origin) form; passing a centre c
    evaluates it for p - c (the bound holds for any c).
    """
    best = 0.0
    for X in (A, B):
        for i in range(0, X.shape[0], _BLOCK):
            Y = np.asarray(X[i:i + _BLOCK], dtype=np.float64)
            if center is not None:
                Y = Y - center[None, :]
            t = Y @ u
            r2 = np.einsum("ij,ij->i", Y, Y) - t * t
            best = max(best, float(np.sqrt(max(r2.max(), 0.0))))
    return best


def subset_full(A: np.ndarray, B: np.ndarray, IA: np.ndarray, IB: np.ndarray) -> float:
    """H^_sf = max(max_{a in A_sel} min_{b in B} ||a-b||, max_{b in B_sel} min_{a in A} ||b-a||)
    (SPEC.md:279 subset-full mode; provably <= H)."""
    ra, _ = row_minima(A, B, rows=IA)
    rb, _ = row_minima(B, A, rows=IB)
    return float(np.sqrt(max(ra.max(), rb.max())))


# ---------------------------------------------------------------- O11 / O12

def paper_parameters(D: int, alpha: float, nX: int) -> tuple[int, int, int]:
    """O11: (m_pc, per-tail count on the centroid axis, per-tail count on each PC).

    Alg. 3 line 1: m = floor(sqrt D), alpha' = alpha/m; Alg. 1/2 (P:205,
    P:242): k_X = max{1, floor(alpha n_X)}. m_pc clamped to >= 1.
    """
    m_pc = max(1, int(np.floor(np.sqrt(D))))
    c0 = max(1, int(np.floor(alpha * nX)))
    c1 = max(1, int(np.floor((alpha / m_pc) * nX)))
    return m_pc, c0, c1


def select_counts(X: np.ndarray, U: np.ndarray, counts: list[int]) -> dict:
    """O6+O7 with a per-direction tail count counts[l] (Alg. 1 uses k_X on the centroid axis,
    Alg. 2 uses floor(alpha' n_X) on the PCs). All of X if 2 counts[l] >= n for any l."""
    n = X.shape[0]
    P = project(X, U)
    lists = [extremes(P[:, l], counts[l]) for l in range(U.shape[1])]
    if any(2 * c >= n for c in counts):
        union = np.arange(n, dtype=np.int64)
    else:
        union = np.unique(np.concatenate([np.concatenate(t) for t in lists])).astype(np.int64)
    return {"lists": lists, "union": union, "proj": P}


def estimate_paper(A: np.ndarray, B: np.ndarray, alpha: float) -> dict:
    """Alg. 3 with the paper's own parameters (O11): m_pc = floor(sqrt D) PCs, alpha on the
    centroid axis (Alg. 1 with alpha), alpha' = alpha/m_pc on each PC (Alg. 2 with alpha')."""
    D = A.shape[1]
    m_pc = min(D, paper_parameters(D, alpha, 1)[0])
    info = directions(A, B, m_pc)
    U = info["U"]
    sel = []
    for X in (A, B):
        _, c0, c1 = paper_parameters(D, alpha, X.shape[0])
        sel.append(select_counts(X, U, [c0] + [c1] * (U.shape[1] - 1)))
    hd = subset_hd(A, B, sel[0]["union"], sel[1]["union"])
    return {"value": hd["value"], "ab": hd["ab"], "ba": hd["ba"], "IA": sel[0]["union"], "IB": sel[1]["union"],
            "size_a": int(sel[0]["union"].size), "size_b": int(sel[1]["union"].size), "U": U,
            "n_dirs": int(U.shape[1]), "k": m_pc}


def sampling_hd(A: np.ndarray, B: np.ndarray, IA: np.ndarray, IB: np.ndarray) -> dict:
    """The paper's sampling baselines given their index draws: exact HD of the samples."""
    return subset_hd(A, B, np.asarray(IA), np.asarray(IB))


def sharded_select(X: np.ndarray, U: np.ndarray, m: int, G: int) -> dict:
    """O12: split rows into G contiguous blocks, local top/bottom-m per block, then
    merge the G*m candidates by the same total order. Must equal `select`."""
    n = X.shape[0]
    P = project(X, U)
    bounds = [(g * n) // G for g in range(G + 1)]
    lists = []
    for l in range(U.shape[1]):
        cb, ct = [], []
        for g in range(G):
            lo, hi = bounds[g], bounds[g + 1]
            if hi <= lo:
                continue
            b, t = extremes(P[lo:hi, l], m)
            cb.append(b + lo)
            ct.append(t + lo)
        cb = np.concatenate(cb)
        ct = np.concatenate(ct)
        mm = min(m, n)
        bo = cb[np.lexsort((cb, P[cb, l]))][:mm]
        to = ct[np.lexsort((ct, -P[ct, l]))][:mm]
        lists.append((bo, to))
    if 2 * m >= n:
        union = np.arange(n, dtype=np.int64)
    else:
        union = np.unique(np.concatenate([np.concatenate(t) for t in lists])).astype(np.int64)
    return {"lists": lists, "union": union}


def sharded_directed_hd(A: np.ndarray, B: np.ndarray, G: int) -> dict:
    """O12 for the exact kernel: rows of A split into G blocks; each block's best
    (d2, lowest row) packed key; the max over blocks must equal directed_hd."""
    n = A.shape[0]
    bounds = [(g * n) // G for g in range(G + 1)]
    best = None
    for g in range(G):
        lo, hi = bounds[g], bounds[g + 1]
        if hi <= lo:
            continue
        r = directed_hd(A[lo:hi], B)
        cand = (r["dist2"], -(r["a"] + lo), r["b"])
        if best is None or cand[:2] > best[:2]:
            best = cand
    return {"dist2": best[0], "dist": float(np.sqrt(best[0])), "a": -best[1], "b": best[2]}
