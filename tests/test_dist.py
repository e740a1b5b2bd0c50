"""World-size-2 gloo tests of the multi-GPU exchange logic (paper_2511_18207_b200/dist.py) on CPU.

The per-rank compute is the oracle's (tests may call it); the product path passes the
CUDA functions. Checks: the sharded max-key all-reduce and witness exchange reproduce
the unsharded oracle result exactly, including the lowest-row tie rule across ranks.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2511_18207_b200.dist import pack_key, row_range, sharded_directed_hd, sharded_hausdorff, unpack_key


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, A, B, q, mode):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = row_range(A.shape[0], rank, world)

    def local_fn(Al, off, Bm):
        rmin, _ = oracle.row_minima(Al, Bm)
        rmin32 = rmin.astype(np.float32)  # the kernel reports fp32 row minima
        i = int(np.argmax(rmin32))
        return pack_key(float(rmin32[i]), off + i)

    def witness_fn(a, Bm):
        rmin, arg = oracle.row_minima(a.reshape(1, -1), Bm)
        return {"b": int(arg[0]), "dist2": float(rmin[0])}

    if mode == "directed":
        r = sharded_directed_hd(A[lo:hi], lo, B, local_fn, witness_fn)
    else:
        r = sharded_hausdorff(A, B, rank, world, lambda Al, off, Bm, c: local_fn(Al, off, Bm), witness_fn)
    q.put((rank, r))
    dist.destroy_process_group()


def _run(A, B, world=2, mode="directed"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, A, B, q, mode)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    return dict(res)


def test_key_packing_orders_like_d2_then_lowest_row():
    k1 = pack_key(2.0, 10)
    k2 = pack_key(2.0, 3)
    k3 = pack_key(2.5, 100)
    assert k3 > k2 > k1
    assert unpack_key(k2) == (2.0, 3)
    assert k3 < 2 ** 63  # non-negative int64 for the NCCL MAX all-reduce


@pytest.mark.parametrize("ties", [False, True])
def test_sharded_equals_unsharded(ties):
    rng = np.random.default_rng(1)
    A = rng.standard_normal((301, 6)).astype(np.float32)
    B = rng.standard_normal((120, 6)).astype(np.float32)
    if ties:  # the global argmax row appears in both shards -> lowest row must win
        ref0 = oracle.directed_hd(A, B)
        A[250] = A[ref0["a"]]
        A[ref0["a"]] = A[ref0["a"]]
    ref = oracle.directed_hd(A, B)
    res = _run(A, B)
    for rank, r in res.items():
        assert r["a"] == ref["a"] and r["b"] == ref["b"], (rank, r, ref)
        assert r["dist2"] == ref["dist2"]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_hausdorff_equals_unsharded(world):
    """Both directions sharded (rows of A for A->B, rows of B for B->A), one MAX all-reduce each:
    the value, both witnesses and the A->B-on-equality rule match the unsharded oracle."""
    rng = np.random.default_rng(5)
    A = rng.standard_normal((157, 5)).astype(np.float32)
    B = (rng.standard_normal((211, 5)) + 0.3).astype(np.float32)
    ref = oracle.hausdorff(A, B)
    for rank, r in _run(A, B, world=world, mode="undirected").items():
        for side in ("ab", "ba"):
            assert (r[side]["a"], r[side]["b"]) == (ref[side]["a"], ref[side]["b"]), (rank, side)
            assert r[side]["dist2"] == ref[side]["dist2"]
        assert r["value"] == ref["value"]
