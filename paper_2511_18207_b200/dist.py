"""Multi-GPU driver: one process per GPU, torch.distributed (NCCL) for the exchange steps.

Sharding (north_star "Shard across one 8xB200 box by rows of A
for the exact kernel, with B replicated and the per-GPU maxima combined by an
NCCL max-allreduce"):

  exact h(A,B)  rank r holds rows [lo_r, hi_r) of A and all of B. Each rank runs
                the fused kernel on its rows and packs its maximum as
                    key = (float_bits(d2) << 32) | (0xFFFFFFFF - global_row)
                (d2 >= 0 so the key is a non-negative int64 and orders like
                (d2, -row)); one all_reduce(MAX) of 8 bytes gives the global
                argmax row with the lowest-row tie rule, bit-identical for any
                rank count. The owner of that row computes the fp64 witness
                column; a second all_reduce shares it.

The compute steps go through the C ABI (Context). `local_fn` / `witness_fn`
exist so the exchange logic can be exercised on CPU ranks (gloo) in tests with
locally computed keys; the product path always passes the CUDA ones.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def row_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous row block of rank `rank` (floor split)."""
    return (n * rank) // world, (n * (rank + 1)) // world


def pack_key(d2: float, row: int) -> int:
    bits = int(np.array([d2], dtype=np.float32).view(np.uint32)[0])
    return (bits << 32) | (0xFFFFFFFF - row)


def unpack_key(key: int) -> tuple[float, int]:
    d2 = float(np.array([key >> 32], dtype=np.uint32).view(np.float32)[0])
    return d2, 0xFFFFFFFF - (key & 0xFFFFFFFF)


def sharded_directed_hd(A_local, row_offset: int, B, local_fn, witness_fn, device=None,
                        group=None) -> dict:
    """h(A,B) with A row-sharded across the group and B replicated.

    local_fn(A_local, row_offset, B) -> packed key of this shard (int)
    witness_fn(a_row, B) -> {"b": int, "dist2": float} (fp64 nearest neighbour)
    """
    key = int(local_fn(A_local, row_offset, B)) if A_local.shape[0] > 0 else 0  # empty shard: no candidate
    t = torch.tensor([key], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    gkey = int(t.item())
    d2_tc, row = unpack_key(gkey)
    nloc = A_local.shape[0]
    mine = row_offset <= row < row_offset + nloc
    w = torch.zeros(2, dtype=torch.float64, device=device)
    if mine:
        r = witness_fn(A_local[row - row_offset], B)
        w[0] = float(r["b"]) + 1.0  # +1 so that "no owner" (0) never wins
        w[1] = r["dist2"]
    dist.all_reduce(w, op=dist.ReduceOp.MAX, group=group)
    b = int(w[0].item()) - 1
    d2 = float(w[1].item())
    return {"dist": float(np.sqrt(d2)), "dist2": d2, "a": row, "b": b, "dist2_tc": d2_tc, "key": gkey}


def sharded_hausdorff(A, B, rank: int, world: int, local_fn, witness_fn, centre=None, device=None,
                      group=None) -> dict:
    """H(A,B) = max(h(A,B), h(B,A)) with both sets replicated on every rank.

    A->B shards the rows of A (B replicated), B->A shards the rows of B (A replicated), each
    side combined by one MAX all-reduce of the packed key plus the witness exchange of
    `sharded_directed_hd`. With `centre` (e.g. prohd_centre(A, B), the centre `hausdorff()`
    uses) both sides prepare their operands about the same point, so the result is
    bit-identical for every rank count. local_fn(A_local, row_offset, B, centre) -> key.
    """
    res = {}
    for side, (R, Cm) in {"ab": (A, B), "ba": (B, A)}.items():
        lo, hi = row_range(R.shape[0], rank, world)
        loc = (lambda A_l, off, Bm: local_fn(A_l, off, Bm, centre))
        res[side] = sharded_directed_hd(R[lo:hi], lo, Cm, loc, witness_fn, device=device, group=group)
    ab, ba = res["ab"], res["ba"]
    value = ab["dist"] if ab["dist2"] >= ba["dist2"] else ba["dist"]  # A->B witness on equality (Q15)
    return {"value": value, "ab": ab, "ba": ba}


def _all_gather_rows(rows: torch.Tensor, D: int, device, group=None) -> torch.Tensor:
    """Concatenate every rank's rows (variable counts) in rank order (C3)."""
    world = dist.get_world_size(group)
    cnt = torch.tensor([rows.shape[0]], dtype=torch.int64, device=device)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt, group=group)
    cnts = [int(c.item()) for c in cnts]
    mx = max(max(cnts), 1)
    pad = torch.zeros(mx, D, dtype=rows.dtype, device=device)
    pad[: rows.shape[0]] = rows
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:c] for b, c in zip(bufs, cnts)], dim=0).contiguous()


def sharded_prohd_estimate(A_local, offA: int, nA: int, B_local, offB: int, nB: int, k: int, m: int,
                           phases, device=None, group=None) -> dict:
    """Alg. 3 with the rows of A and B sharded across the group.

    Rank r holds rows [offA, offA + len(A_local)) of A and [offB, ...) of B (contiguous
    blocks in rank order; rank 0 starts at row 0). `phases` provides the per-rank compute
    (CUDA: `CudaPhases(ctx)`): shift, local_moments, directions, local_candidates,
    merge_union, gather_owned, local_fn, witness_fn. Collectives: broadcast of the shift,
    C0 MAX all-reduce of the column ranges (int8 Gram; skipped when local_colmax returns None),
    C1 SUM all-reduce of the moments, C2 all-gather of the candidate lists, C3 all-gather
    of the selected rows, C4 MAX all-reduce of the subset-HD keys.
    """
    rank = dist.get_rank(group)
    D = A_local.shape[1]
    # shift from the first <= 4096 rows (owned by rank 0), broadcast
    s = torch.zeros(D, dtype=torch.float64, device=device)
    if rank == 0:
        s.copy_(torch.as_tensor(phases.shift(A_local[:4096], B_local[:4096])))
    dist.broadcast(s, src=0, group=group)
    s_np = s.cpu().numpy()
    # C0 (int8 Gram): MAX all-reduce of the per-feature ranges, so every rank quantises on the
    # same fixed-point grid; C1: SUM all-reduce of the moments
    colmax = phases.local_colmax(A_local, B_local, s_np)
    if colmax is not None:
        dist.all_reduce(colmax, op=dist.ReduceOp.MAX, group=group)
    mom = phases.local_moments(A_local, B_local, s_np, colmax)
    dist.all_reduce(mom, op=dist.ReduceOp.SUM, group=group)
    dirs, n_dirs = phases.directions(mom, nA, nB, D, k, s_np)
    # C2 + merge + C3 per set
    world = dist.get_world_size(group)
    unions, subsets = [], []
    for X_local, off, n in ((A_local, offA, nA), (B_local, offB, nB)):
        val, idx = phases.local_candidates(X_local, off, dirs, m)
        vals = [torch.empty_like(val) for _ in range(world)]
        idxs = [torch.empty_like(idx) for _ in range(world)]
        dist.all_gather(vals, val, group=group)
        dist.all_gather(idxs, idx, group=group)
        union = phases.merge_union(torch.stack(vals), torch.stack(idxs), m, n)
        rows, _, _ = phases.gather_owned(X_local, off, union)
        subsets.append(_all_gather_rows(rows, D, device, group))
        unions.append(union)
    # C4: exact HD on the subsets, rows of each subset sharded over the ranks; every rank
    # prepares the distance operands about the same centre(A_sel, B_sel) as prohd_estimate
    centre = phases.centre(subsets[0], subsets[1])
    res = {}
    for side, (R, Cm, uR, uC) in {"ab": (subsets[0], subsets[1], unions[0], unions[1]),
                                  "ba": (subsets[1], subsets[0], unions[1], unions[0])}.items():
        lo, hi = row_range(R.shape[0], rank, world)
        local = (lambda A_l, off, Bm: phases.local_fn(A_l, off, Bm, centre))
        r = sharded_directed_hd(R[lo:hi], lo, Cm, local, phases.witness_fn, device=device, group=group)
        res[side] = {**r, "a": int(uR[r["a"]].item()), "b": int(uC[r["b"]].item())}
    ab, ba = res["ab"], res["ba"]
    value = ab["dist"] if ab["dist2"] >= ba["dist2"] else ba["dist"]
    return {"value": value, "ab": ab, "ba": ba, "size_a": int(unions[0].numel()),
            "size_b": int(unions[1].numel()), "n_dirs": n_dirs, "IA": unions[0], "IB": unions[1], "U": dirs}


class CudaPhases:
    """The product phase implementations: every step runs in libprohd.so kernels."""

    def __init__(self, ctx, dmma: bool = False):
        self.ctx = ctx
        self.dmma = dmma  # True: the fp64 DMMA Gram for the moments (one-shot option k1_path = 0)
        self.local_fn, self.witness_fn = cuda_fns(ctx)

    def shift(self, A_first, B_first):
        return self.ctx.shift(A_first, B_first)

    def centre(self, X, Y):
        return self.ctx.centre(X, Y)

    def local_colmax(self, A_local, B_local, s):
        """Column ranges for the int8 Gram (D <= 256, D % 4 == 0), else None (fp64 DMMA Gram)."""
        D = A_local.shape[1]
        if D > 256 or D % 4 != 0 or self.dmma:
            return None
        return self.ctx.local_colmax(A_local, B_local, s)

    def local_moments(self, A_local, B_local, s, colmax=None):
        if colmax is None:
            return self.ctx.local_moments(A_local, B_local, s)
        return self.ctx.local_moments_i8(A_local, B_local, s, colmax)

    def directions(self, moments, nA, nB, D, k, s):
        return self.ctx.directions(moments, nA, nB, D, k, s)

    def local_candidates(self, X_local, off, dirs, m):
        return self.ctx.local_candidates(X_local, off, dirs, m)

    def merge_union(self, vals, idxs, m, n):
        return self.ctx.merge_union(vals, idxs, m, n)

    def gather_owned(self, X_local, off, union):
        return self.ctx.gather_owned(X_local, off, union)


def cuda_fns(ctx):
    """The product local/witness functions: both run in libprohd.so kernels."""
    def local_fn(A_local, row_offset, B, centre=None):
        return ctx.directed_hd_local(A_local, row_offset, B, centre)

    def witness_fn(a_row, B):
        return ctx.directed_hd_witness(a_row, B)

    return local_fn, witness_fn
