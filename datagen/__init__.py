"""Seeded synthetic workloads for the ProHD hot path (BASELINE.json `configs`).

This module is the ONE piece shared by the oracle (`oracle/`) and the CUDA path
(`paper_2511_18207_b200/`). It holds no part of the method's arithmetic: it only
draws point clouds. Every recipe is frozen here and restated in DESIGN.md
("Input recipe"); SURVEY.md §8(d2) is the source of the shapes/distributions.

Stand-ins: the paper measures on CIFAR-10 / MNIST (after PCA), Higgs and uniform
random clouds. None of those datasets is in this container,
so these five synthetic designs (BASELINE.json configs 1-5) stand in for them;
nothing here reproduces any record of those datasets.

Rules
-----
* All draws are float64 from numpy PCG64, then cast to float32 (round to nearest
  even); the cast arrays are what both sides read.
* cfg1 is literal: ``rng = default_rng(seed)``, A drawn then B (BASELINE.json cfg1,
  seed 0; SURVEY.md §8(c3) pins the sha256 of these bytes).
* cfg2-cfg5: shared parameters come from ``default_rng([cfg, seed, 2])``; row
  chunk c (``CHUNK`` rows) of A is drawn from ``default_rng([cfg, seed, 0, c])``
  and of B from ``default_rng([cfg, seed, 1, c])``, each chunk drawing its
  variables in the order listed per recipe. Independent chunk streams keep host
  memory bounded and let chunks (and A and B) be generated in parallel.
* ``rows=(lo, hi)`` generates only that row range of a set bit-identically to the
  full draw (used for row-sharded multi-GPU runs and for oracle samples).
"""
from __future__ import annotations

import hashlib
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

CHUNK = 65536


@dataclass(frozen=True)
class Config:
    cfg: int
    name: str
    n: int
    D: int
    k: int
    frac: float  # per-direction tail size m = max(1, floor(frac * n)); cfg1 uses m_abs
    m_abs: int | None = None

    def m(self, n: int | None = None) -> int:
        """Per-(set, direction, tail) count m (floor + clamp)."""
        if self.m_abs is not None:
            return self.m_abs
        nn = self.n if n is None else n
        return max(1, int(np.floor(self.frac * nn)))


CONFIGS = {
    1: Config(1, "tiny", 2000, 16, 4, 0.0, m_abs=20),
    2: Config(2, "clustered", 100_000, 64, 8, 0.005),
    3: Config(3, "embedding-drift", 500_000, 128, 8, 0.002),
    4: Config(4, "image-like", 1_000_000, 256, 16, 0.001),
    5: Config(5, "heavy-tailed", 2_000_000, 256, 16, 0.0005),
}


def sha256(x: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def _haar(rng: np.random.Generator, D: int) -> np.ndarray:
    g = rng.standard_normal((D, D))
    q, r = np.linalg.qr(g)
    return q * np.sign(np.diag(r))[None, :]


# ----------------------------------------------------------------------------
# shared (per-config) parameters
# ----------------------------------------------------------------------------

def _params(cfg: int, seed: int, D: int) -> dict:
    rng = np.random.default_rng([cfg, seed, 2])
    p: dict = {}
    if cfg == 2:
        p["mu"] = 5.0 * rng.standard_normal((10, D))
        p["sigma"] = rng.uniform(0.5, 2.0, size=10)
        p["mu_b"] = p["mu"] + 0.5 * rng.standard_normal((10, D))
    elif cfg == 3:
        lam = np.arange(1, D + 1, dtype=np.float64) ** -1.2
        Q = _haar(rng, D)
        partners = rng.choice(np.arange(8, D), size=8, replace=False)
        th = np.deg2rad(10.0)
        QB = Q.copy()
        for i in range(8):
            qi, qp = QB[:, i].copy(), QB[:, partners[i]].copy()
            QB[:, i] = np.cos(th) * qi + np.sin(th) * qp
            QB[:, partners[i]] = -np.sin(th) * qi + np.cos(th) * qp
        w = rng.standard_normal(D)
        p["sqrt_lam"] = np.sqrt(lam)
        p["Q"] = Q
        p["QB"] = QB
        p["drift"] = 0.05 * w / np.linalg.norm(w)
    elif cfg == 4:
        r = 32
        VA = np.abs(rng.standard_normal((r, D)))
        VB = VA.copy()
        VB[24:32] = np.abs(rng.standard_normal((8, D)))
        p["VA"], p["VB"], p["s"] = VA, VB, np.pi / 128.0
    elif cfg == 5:
        lam = 10.0 ** rng.uniform(-2.0, 1.0, size=D)
        Q = _haar(rng, D)
        G = rng.standard_normal((D, D))
        K = G - G.T
        K = K / np.linalg.norm(K, 2)
        th = 0.02
        I = np.eye(D)
        R = np.linalg.solve(I - th * K / 2, I + th * K / 2)
        p["sqrt_lam"] = np.sqrt(lam)
        p["Q"] = Q
        p["QB"] = R @ Q
    return p


def _chunk(cfg: int, which: int, rng: np.random.Generator, rows: int, D: int,
           p: dict, gstart: int, outliers: np.ndarray | None) -> np.ndarray:
    """Draw `rows` rows of set `which` (0=A, 1=B) in float64."""
    if cfg == 2:
        lab = rng.integers(0, 10, size=rows)
        mu = p["mu"] if which == 0 else p["mu_b"]
        x = mu[lab] + p["sigma"][lab][:, None] * rng.standard_normal((rows, D))
        if which == 1 and outliers is not None:
            sel = outliers[(outliers >= gstart) & (outliers < gstart + rows)] - gstart
            u = rng.uniform(-20.0, 20.0, size=(sel.size, D))
            x[sel] = u
        return x
    if cfg == 3:
        z = rng.standard_normal((rows, D)) * p["sqrt_lam"][None, :]
        x = z @ (p["Q"] if which == 0 else p["QB"]).T
        if which == 1:
            x = x + p["drift"][None, :]
        return x / np.linalg.norm(x, axis=1, keepdims=True)
    if cfg == 4:
        V = p["VA"] if which == 0 else p["VB"]
        u = np.abs(rng.standard_normal((rows, V.shape[0])))
        e = 0.02 * rng.standard_normal((rows, D))
        return np.clip(p["s"] * (u @ V) + e, 0.0, 1.0)
    if cfg == 5:
        z = rng.standard_normal((rows, D)) * p["sqrt_lam"][None, :]
        w = rng.chisquare(3.0, size=rows)
        x = (z @ (p["Q"] if which == 0 else p["QB"]).T) / np.sqrt(w / 3.0)[:, None]
        if which == 1:
            x = x + 0.3
        return x
    raise ValueError(cfg)


def generate_set(cfg: int, which: str, seed: int = 0, n: int | None = None,
                 rows: tuple[int, int] | None = None) -> np.ndarray:
    """Return set `which` ('A' or 'B') of config `cfg` as C-contiguous float32.

    `n` overrides the config's size (reduced-scale parity cases use the same
    recipe with a smaller n). `rows=(lo, hi)` returns only that row range.
    """
    c = CONFIGS[cfg]
    n = c.n if n is None else n
    D = c.D
    w = {"A": 0, "B": 1}[which]
    lo, hi = (0, n) if rows is None else rows
    if not (0 <= lo <= hi <= n):
        raise ValueError("bad row range")
    if cfg == 1:
        rng = np.random.default_rng(seed)
        a = rng.standard_normal((n, D))
        if w == 0:
            return np.ascontiguousarray(a[lo:hi].astype(np.float32))
        b = rng.standard_normal((n, D))
        b[:, 0] += 0.5
        return np.ascontiguousarray(b[lo:hi].astype(np.float32))
    p = _params(cfg, seed, D)
    outliers = None
    if cfg == 2 and w == 1:
        orng = np.random.default_rng([cfg, seed, 3])
        outliers = np.sort(orng.choice(n, size=n // 1000, replace=False))
    out = np.empty((hi - lo, D), dtype=np.float32)

    def work(c: int) -> None:
        g = c * CHUNK
        r = min(CHUNK, n - g)
        rng = np.random.default_rng([cfg, seed, w, c])
        x = _chunk(cfg, w, rng, r, D, p, g, outliers)
        s0, s1 = max(lo, g), min(hi, g + r)
        out[s0 - lo:s1 - lo] = x[s0 - g:s1 - g].astype(np.float32)

    chunks = list(range(lo // CHUNK, (hi + CHUNK - 1) // CHUNK)) if hi > lo else []
    if len(chunks) <= 1:
        for c in chunks:
            work(c)
    else:
        with ThreadPoolExecutor(max_workers=min(len(chunks), os.cpu_count() or 1)) as ex:
            list(ex.map(work, chunks))
    return out


def generate(cfg: int, seed: int = 0, n: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """(A, B) for config `cfg` at size n (default: the config's n)."""
    return generate_set(cfg, "A", seed, n), generate_set(cfg, "B", seed, n)


def sample_rows(n: int, count: int, seed: int = 12345) -> np.ndarray:
    """Seeded uniform sample of `count` distinct row indices of [0, n), sorted."""
    rng = np.random.default_rng([99, seed])
    count = min(count, n)
    return np.sort(rng.choice(n, size=count, replace=False))


# ----------------------------------------------------------------------------
# Paper workloads and baseline draws
# ----------------------------------------------------------------------------

def random_clouds(nA: int, nB: int, D: int, seed: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """PAPER.md:457 "randomly generated point clouds which are distributed uniformly in the
    unit cube [0,1]^D with an offset of 0.1": A ~ U[0,1]^D, B ~ U[0,1]^D + 0.1 (the offset
    applied to B, SPEC.md:391-399 reading), float64 draws cast to float32."""
    rng = np.random.default_rng([7, seed, D])
    A = rng.uniform(0.0, 1.0, size=(nA, D))
    B = rng.uniform(0.0, 1.0, size=(nB, D)) + 0.1
    return A.astype(np.float32), B.astype(np.float32)


def uniform_sample(n: int, size: int, seed: int) -> np.ndarray:
    """Random Sampling baseline draw: `size` indices of [0, n) uniformly
    without replacement (sorted)."""
    rng = np.random.default_rng([11, seed, n])
    return np.sort(rng.choice(n, size=min(size, n), replace=False)).astype(np.int64)


def systematic_sample(n: int, alpha: float, seed: int) -> np.ndarray:
    """Systematic Random Sampling draw: a seeded random permutation of [0, n),
    then every floor(1/alpha)-th element starting at position 0."""
    stride = int(np.floor(1.0 / alpha))
    if stride < 1:
        raise ValueError("alpha must be <= 1")
    rng = np.random.default_rng([13, seed, n])
    perm = rng.permutation(n)
    return perm[::stride].astype(np.int64)
