"""World-size-2 gloo test of the sharded ProHD driver (dist.sharded_prohd_estimate) on CPU.

The per-rank phases are implemented here with the oracle's arithmetic (OraclePhases, tests
only); the product passes dist.CudaPhases. The sharded result must equal the single-process
oracle estimate exactly (same directions up to rounding, same unions, same witnesses).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from oracle import prohd as OP
from paper_2511_18207_b200.dist import pack_key, row_range, sharded_prohd_estimate


class OraclePhases:
    def shift(self, Af, Bf):
        X = np.concatenate([np.asarray(Af, np.float64), np.asarray(Bf, np.float64)])
        return X.mean(axis=0)

    def local_colmax(self, A_l, B_l, s):
        return None  # no fixed-point grid: fp64 moments

    def local_moments(self, A_l, B_l, s, colmax=None):
        A = np.asarray(A_l, np.float64) - s
        B = np.asarray(B_l, np.float64) - s
        G = A.T @ A + B.T @ B
        return torch.from_numpy(np.concatenate([A.sum(0), B.sum(0), G.ravel()]))

    def directions(self, mom, nA, nB, D, k, s):
        mom = mom.numpy()
        SA, SB, G = mom[:D], mom[D:2 * D], mom[2 * D:].reshape(D, D)
        d = SB / nB - SA / nA
        nrm = np.linalg.norm(d)
        u0 = d / nrm if nrm >= 1e-9 else np.eye(D)[0]
        ms = (SA + SB) / (nA + nB)
        C = G / (nA + nB) - np.outer(ms, ms)
        _, V = OP.top_components(0.5 * (C + C.T), k) if k > 0 else (None, np.zeros((D, 0)))
        U = np.concatenate([u0[:, None], V], axis=1)
        return torch.from_numpy(np.ascontiguousarray(U.T)), U.shape[1]

    def local_candidates(self, X_l, off, dirs, m):
        P = np.asarray(X_l, np.float64) @ dirs.numpy().T
        nd = dirs.shape[0]
        val = np.zeros((nd, 2, m))
        idx = -np.ones((nd, 2, m), np.int64)
        for l in range(nd):
            if P.shape[0] == 0:
                continue
            b, t = OP.extremes(P[:, l], m)
            for ti, lst in ((0, t), (1, b)):
                val[l, ti, :len(lst)] = P[lst, l]
                idx[l, ti, :len(lst)] = lst + off
        return torch.from_numpy(val), torch.from_numpy(idx)

    def merge_union(self, vals, idxs, m, n):
        if 2 * m >= n:
            return torch.arange(n)
        vals, idxs = vals.numpy(), idxs.numpy()
        keep = []
        for l in range(vals.shape[1]):
            for t in range(2):
                v = vals[:, l, t].ravel()
                i = idxs[:, l, t].ravel()
                ok = i >= 0
                v, i = v[ok], i[ok]
                order = np.lexsort((i, -v if t == 0 else v))[:m]
                keep.append(i[order])
        return torch.from_numpy(np.unique(np.concatenate(keep)))

    def gather_owned(self, X_l, off, union):
        u = union.numpy()
        sel = u[(u >= off) & (u < off + X_l.shape[0])] - off
        return torch.as_tensor(np.asarray(X_l)[sel]), 0, len(sel)

    def centre(self, X, Y):
        return None  # the oracle's distances are exact: no translation needed

    def local_fn(self, Al, off, Bm, centre=None):
        rmin, _ = oracle.row_minima(np.asarray(Al), np.asarray(Bm))
        rmin32 = rmin.astype(np.float32)
        i = int(np.argmax(rmin32))
        return pack_key(float(rmin32[i]), off + i)

    def witness_fn(self, a, Bm):
        rmin, arg = oracle.row_minima(np.asarray(a).reshape(1, -1), np.asarray(Bm))
        return {"b": int(arg[0]), "dist2": float(rmin[0])}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, A, B, k, m, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    la, ha = row_range(A.shape[0], rank, world)
    lb, hb = row_range(B.shape[0], rank, world)
    r = sharded_prohd_estimate(torch.from_numpy(A[la:ha]), la, A.shape[0], torch.from_numpy(B[lb:hb]), lb,
                               B.shape[0], k, m, OraclePhases())
    q.put((rank, {"value": r["value"], "ab": r["ab"], "ba": r["ba"], "IA": r["IA"].numpy(),
                  "IB": r["IB"].numpy(), "n_dirs": r["n_dirs"]}))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_prohd_equals_oracle(world):
    rng = np.random.default_rng(world)
    A = (rng.standard_normal((523, 6)) * [3, 2, 1, 1, 0.5, 0.2]).astype(np.float32)
    B = (rng.standard_normal((411, 6)) + 0.3).astype(np.float32)
    k, m = 3, 9
    ref = OP.estimate(A, B, k, m)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, A, B, k, m, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=180) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for rank, r in res.items():
        assert np.array_equal(r["IA"], ref["IA"]) and np.array_equal(r["IB"], ref["IB"]), rank
        assert r["value"] == ref["value"]
        assert (r["ab"]["a"], r["ab"]["b"]) == (ref["ab"]["a"], ref["ab"]["b"])
        assert (r["ba"]["a"], r["ba"]["b"]) == (ref["ba"]["a"], ref["ba"]["b"])
        assert r["n_dirs"] == ref["n_dirs"]
