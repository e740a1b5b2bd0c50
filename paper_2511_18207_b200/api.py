"""Python binding of the C ABI (include/prohd.h): same names, argument marshalling only.

Every step of the path runs in libprohd.so's sm_100a kernels. PyTorch supplies
device memory (inputs, the workspace) and the CUDA stream. There is no CPU
fallback: without the library or a B200 these calls raise.

Inputs are 2-D float32 tensors (n x D, contiguous). CUDA tensors are passed as
device pointers; CPU tensors are passed as host pointers and the library copies
them to the device inside the call (the end-to-end path).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib as L


class ProHDError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{L.STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


def _directed(d: L.Directed) -> dict:
    return {"dist": d.dist, "dist2": d.dist2, "a": int(d.a), "b": int(d.b), "dist2_tc": d.dist2_tc}


def _as_points(X, name: str) -> torch.Tensor:
    if isinstance(X, np.ndarray):
        X = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32))
    if not isinstance(X, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor or numpy array")
    if X.dtype != torch.float32 or X.dim() != 2:
        raise TypeError(f"{name} must be a 2-D float32 tensor (got {X.dtype}, dim {X.dim()})")
    return X.contiguous()


class Context:
    """A prohd_ctx bound to one CUDA device, with a torch-allocated workspace."""

    def __init__(self, device: int | None = None):
        self.lib = L.load()
        if device is None:
            device = torch.cuda.current_device()
        self.device = int(device)
        h = C.c_void_p()
        rc = self.lib.prohd_create(self.device, None, C.byref(h))
        if rc != L.PROHD_OK:
            raise ProHDError(rc, f"prohd_create(device={self.device}) failed")
        self.h = h
        self._ws = None

    def close(self):
        if getattr(self, "h", None):
            self.lib.prohd_destroy(self.h)
            self.h = None

    __del__ = close

    # ---------------------------------------------------------------- plumbing
    def _check(self, rc: int):
        if rc != L.PROHD_OK:
            raise ProHDError(rc, self.lib.prohd_last_error(self.h).decode())

    def reserve(self, nA: int, nB: int, D: int, k: int = 0, m: int = 1, host_inputs: bool = False,
                certified: bool = False) -> int:
        flags = (L.PROHD_WS_HOST_INPUTS if host_inputs else 0) | (L.PROHD_WS_CERTIFIED if certified else 0)
        need = int(self.lib.prohd_workspace_bytes(nA, nB, D, k, m, flags))
        return self._ensure_ws(need)

    def _ensure_ws(self, need: int) -> int:
        if self._ws is None or self._ws.numel() < need:
            self._ws = None
            torch.cuda.synchronize(self.device)
            self._ws = torch.empty(need, dtype=torch.uint8, device=f"cuda:{self.device}")
        self._check(self.lib.prohd_set_workspace(self.h, self._ws.data_ptr(), self._ws.numel()))
        return need

    def _prepare(self, A, B, k=0, m=1, certified=False):
        A = _as_points(A, "A")
        B = _as_points(B, "B")
        if A.shape[1] != B.shape[1]:
            raise ValueError("A and B must have the same dimension D")
        host = not (A.is_cuda and B.is_cuda)
        self.reserve(A.shape[0], B.shape[0], A.shape[1], k, m, host_inputs=host, certified=certified)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        self._check(self.lib.prohd_set_stream(self.h, C.c_void_p(stream)))
        return A, B

    def launch_count(self) -> int:
        """prohd_launch_count: kernels this process has launched through the library."""
        v = C.c_int64(0)
        self._check(self.lib.prohd_launch_count(C.byref(v)))
        return int(v.value)

    def enable_timing(self, on: bool = True):
        """Record per-phase CUDA events inside every following call (prohd_enable_timing)."""
        self._check(self.lib.prohd_enable_timing(self.h, 1 if on else 0))

    def last_timings(self) -> dict:
        """Per-phase device milliseconds and kernel-launch counts of the last call."""
        t = L.Timings()
        self._check(self.lib.prohd_last_timings(self.h, C.byref(t)))
        return {name: getattr(t, name) for name, _ in L.Timings._fields_}

    # ---------------------------------------------------------------- ABI calls
    def directed_hd(self, A, B) -> dict:
        A, B = self._prepare(A, B)
        out = L.Directed()
        self._check(self.lib.directed_hd(self.h, A.data_ptr(), A.shape[0], B.data_ptr(), B.shape[0],
                                         A.shape[1], C.byref(out)))
        return _directed(out)

    def hausdorff(self, A, B) -> dict:
        A, B = self._prepare(A, B)
        out = L.HD()
        self._check(self.lib.hausdorff(self.h, A.data_ptr(), A.shape[0], B.data_ptr(), B.shape[0],
                                       A.shape[1], C.byref(out)))
        return {"value": out.value, "ab": _directed(out.ab), "ba": _directed(out.ba)}

    def covariance(self, A, B):
        """prohd_covariance (test hook): (mu, C, path) of step 1a, path 1 = int8 Gram, 0 = DMMA."""
        A, B = self._prepare(A, B, 0, 1)
        D = A.shape[1]
        mu = np.empty(D, np.float64)
        Cm = np.empty((D, D), np.float64)
        path = C.c_int32(0)
        self._check(self.lib.prohd_covariance(self.h, A.data_ptr(), A.shape[0], B.data_ptr(), B.shape[0], D,
                                              mu.ctypes.data, Cm.ctypes.data, C.byref(path)))
        return mu, Cm, int(path.value)

    def hausdorff_minima(self, A, B):
        """hausdorff() plus both directions' per-row minima (test hook): (result, rowmin, colmin)."""
        A, B = self._prepare(A, B)
        dev = f"cuda:{self.device}"
        rowmin = torch.empty(A.shape[0], dtype=torch.float32, device=dev)
        colmin = torch.empty(B.shape[0], dtype=torch.float32, device=dev)
        out = L.HD()
        self._check(self.lib.hausdorff_minima(self.h, A.data_ptr(), A.shape[0], B.data_ptr(), B.shape[0], A.shape[1],
                                              rowmin.data_ptr(), colmin.data_ptr(), C.byref(out)))
        return ({"value": out.value, "ab": _directed(out.ab), "ba": _directed(out.ba)}, rowmin, colmin)

    def directed_hd_rowmin(self, A, B) -> torch.Tensor:
        A, B = self._prepare(A, B)
        rowmin = torch.empty(A.shape[0], dtype=torch.float32, device=f"cuda:{self.device}")
        self._check(self.lib.directed_hd_rowmin(self.h, A.data_ptr(), A.shape[0], B.data_ptr(), B.shape[0],
                                                A.shape[1], rowmin.data_ptr()))
        return rowmin

    def _est_out(self, out: L.Est) -> dict:
        return {"value": out.value, "ab": _directed(out.ab), "ba": _directed(out.ba),
                "size_a": int(out.size_a), "size_b": int(out.size_b), "n_dirs": int(out.n_dirs)}

    def prohd_estimate(self, A, B, k: int, m: int, return_dirs: bool = False,
                       return_indices: bool = False, certified: bool = False) -> dict:
        """Alg. 3; certified=True gives the subset-full estimate (prohd_estimate_certified)."""
        A, B = self._prepare(A, B, k, m, certified=certified)
        nA, nB, D = A.shape[0], B.shape[0], A.shape[1]
        out = L.Est()
        dirs = np.zeros((k + 1, D), dtype=np.float64) if return_dirs else None
        capA = min(nA, 2 * m * (k + 1))
        capB = min(nB, 2 * m * (k + 1))
        ia = np.empty(capA, dtype=np.int64) if return_indices else None
        ib = np.empty(capB, dtype=np.int64) if return_indices else None
        ptr = (lambda a: a.ctypes.data if a is not None else None)
        fn = self.lib.prohd_estimate_certified if certified else self.lib.prohd_estimate
        self._check(fn(self.h, A.data_ptr(), nA, B.data_ptr(), nB, D, k, m, C.byref(out), ptr(dirs), ptr(ia),
                       ptr(ib)))
        res = self._est_out(out)
        if return_dirs:
            res["U"] = dirs[: res["n_dirs"]].T.copy()  # D x n_dirs
        if return_indices:
            res["IA"] = ia[: res["size_a"]].copy()
            res["IB"] = ib[: res["size_b"]].copy()
        return res

    def prohd_estimate_alpha(self, A, B, alpha: float, return_dirs: bool = False,
                             return_indices: bool = False) -> dict:
        """Paper-literal Alg. 3: k = floor(sqrt D) PCs, alpha on the centroid axis, alpha/k on the PCs."""
        A0, B0 = _as_points(A, "A"), _as_points(B, "B")
        nA, nB, D = A0.shape[0], B0.shape[0], A0.shape[1]
        k = min(D, max(1, int(np.floor(np.sqrt(D)))))
        c = [max(1, int(np.floor(alpha * x))) for x in (nA, nB)] + \
            [max(1, int(np.floor((alpha / k) * x))) for x in (nA, nB)]
        mmax = max(c)
        A, B = self._prepare(A0, B0, k, mmax)
        out = L.Est()
        dirs = np.zeros((k + 1, D), dtype=np.float64) if return_dirs else None
        capA = min(nA, 2 * mmax * (k + 1))
        capB = min(nB, 2 * mmax * (k + 1))
        ia = np.empty(capA, dtype=np.int64) if return_indices else None
        ib = np.empty(capB, dtype=np.int64) if return_indices else None
        ptr = (lambda a: a.ctypes.data if a is not None else None)
        self._check(self.lib.prohd_estimate_alpha(self.h, A.data_ptr(), nA, B.data_ptr(), nB, D, float(alpha),
                                                  C.byref(out), ptr(dirs), ptr(ia), ptr(ib)))
        res = self._est_out(out)
        if return_dirs:
            res["U"] = dirs[: res["n_dirs"]].T.copy()
        if return_indices:
            res["IA"] = ia[: res["size_a"]].copy()
            res["IB"] = ib[: res["size_b"]].copy()
        return res

    def hausdorff_subsets(self, A, idxA, B, idxB) -> dict:
        """H(A[idxA], B[idxB]) with witnesses as indices into A and B."""
        A, B = self._prepare(A, B)
        ia = np.ascontiguousarray(np.asarray(idxA, dtype=np.int64))
        ib = np.ascontiguousarray(np.asarray(idxB, dtype=np.int64))
        self.reserve(max(A.shape[0], B.shape[0]), max(A.shape[0], B.shape[0]), A.shape[1],
                     host_inputs=not (A.is_cuda and B.is_cuda))
        out = L.HD()
        self._check(self.lib.hausdorff_subsets(self.h, A.data_ptr(), A.shape[0], ia.ctypes.data, ia.size,
                                               B.data_ptr(), B.shape[0], ib.ctypes.data, ib.size, A.shape[1],
                                               C.byref(out)))
        return {"value": out.value, "ab": _directed(out.ab), "ba": _directed(out.ba)}

    def bounds(self, A, B, U: np.ndarray) -> dict:
        """f2 bound report for directions U (D x n_dirs): per-direction delta (origin, centred),
        h_u(A,B), h_u(B,A); H_U, min delta and H_U + 2 min delta (Eq. 4)."""
        U = np.asarray(U, dtype=np.float64)
        n_dirs = U.shape[1]
        A, B = self._prepare(A, B)
        nmax = max(A.shape[0], B.shape[0])
        D = A.shape[1]
        extra = 8 * (4 * n_dirs * nmax + 256 * n_dirs * (nmax // 1024 + 1) + 2 * 296 * D) + (1 << 20)
        self._ensure_ws(self._ws.numel() + extra if self._ws is not None else extra)
        dirs = np.ascontiguousarray(U.T)
        per = np.zeros((n_dirs, 4), dtype=np.float64)
        summ = np.zeros(3, dtype=np.float64)
        self._check(self.lib.prohd_bounds(self.h, A.data_ptr(), A.shape[0], B.data_ptr(), B.shape[0], D,
                                          dirs.ctypes.data, n_dirs, per.ctypes.data, summ.ctypes.data))
        return {"delta_origin": per[:, 0].copy(), "delta_centered": per[:, 1].copy(), "hu_ab": per[:, 2].copy(),
                "hu_ba": per[:, 3].copy(), "H_U": summ[0], "min_delta": summ[1], "upper": summ[2]}

    def prohd_estimate_with_dirs(self, A, B, U: np.ndarray, m: int, return_indices: bool = True) -> dict:
        U = np.asarray(U, dtype=np.float64)
        n_dirs = U.shape[1]
        A, B = self._prepare(A, B, n_dirs - 1, m)
        nA, nB, D = A.shape[0], B.shape[0], A.shape[1]
        dirs = np.ascontiguousarray(U.T)  # [n_dirs][D]
        out = L.Est()
        capA = min(nA, 2 * m * n_dirs)
        capB = min(nB, 2 * m * n_dirs)
        ia = np.empty(capA, dtype=np.int64)
        ib = np.empty(capB, dtype=np.int64)
        self._check(self.lib.prohd_estimate_with_dirs(self.h, A.data_ptr(), nA, B.data_ptr(), nB, D, n_dirs, m,
                                                      dirs.ctypes.data, C.byref(out), ia.ctypes.data,
                                                      ib.ctypes.data))
        res = self._est_out(out)
        res["IA"] = ia[: res["size_a"]].copy()
        res["IB"] = ib[: res["size_b"]].copy()
        return res

    def directed_hd_local(self, A_local, row_offset: int, B, centre=None) -> int:
        """Packed key of this row shard; `centre` (fp64, D) defaults to centre(-, B)."""
        A, B = self._prepare(A_local, B)
        key = C.c_uint64()
        cptr = None
        if centre is not None:
            c = centre if isinstance(centre, torch.Tensor) else torch.as_tensor(np.asarray(centre, np.float64))
            c = c.to(dtype=torch.float64).contiguous()
            cptr = c.data_ptr()
        self._check(self.lib.directed_hd_local(self.h, A.data_ptr(), A.shape[0], int(row_offset), B.data_ptr(),
                                               B.shape[0], A.shape[1], cptr, C.byref(key)))
        return int(key.value)

    def centre(self, X, Y) -> np.ndarray:
        """prohd_centre: fp64 mean of the first <= 4096 rows of X and of Y (device tensors)."""
        X, Y = _as_points(X, "X"), _as_points(Y, "Y")
        D = X.shape[1]
        self._shard_ws(max(X.shape[0], Y.shape[0]), 1, D, 0, 1)
        out = np.zeros(D, dtype=np.float64)
        self._check(self.lib.prohd_centre(self.h, X.data_ptr(), X.shape[0], Y.data_ptr(), Y.shape[0], D,
                                          out.ctypes.data))
        return out

    def project(self, X, dirs):
        """prohd_project (test hook): fp32 projections (L x n, device tensor) of the device
        points X onto the fp64 directions dirs (L x D) and the bound eps on their error."""
        X = _as_points(X, "X")
        dirs = torch.as_tensor(dirs, dtype=torch.float64).to(X.device).contiguous()
        Ld, D = dirs.shape
        self._ensure_ws(Ld * D * 4 + 1024)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        self._check(self.lib.prohd_set_stream(self.h, C.c_void_p(stream)))
        P = torch.empty((Ld, X.shape[0]), dtype=torch.float32, device=X.device)
        eps = C.c_double(0.0)
        self._check(self.lib.prohd_project(self.h, X.data_ptr(), X.shape[0], D, dirs.data_ptr(), Ld,
                                           P.data_ptr(), C.byref(eps)))
        return P, eps.value

    def directed_hd_witness(self, a, B) -> dict:
        a = _as_points(a.reshape(1, -1) if a.dim() == 1 else a, "a")
        a, B = self._prepare(a, B)
        out = L.Directed()
        self._check(self.lib.directed_hd_witness(self.h, a.data_ptr(), B.data_ptr(), B.shape[0], B.shape[1],
                                                 C.byref(out)))
        return _directed(out)


    # ---------------------------------------------------------------- sharded ProHD phases
    def _shard_ws(self, n_local: int, n_total: int, D: int, k: int, m: int):
        need = int(self.lib.prohd_shard_workspace_bytes(n_local, n_total, D, k, m, 0))
        self._ensure_ws(need)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        self._check(self.lib.prohd_set_stream(self.h, C.c_void_p(stream)))

    def shift(self, A_first, B_first) -> np.ndarray:
        A, B = _as_points(A_first, "A"), _as_points(B_first, "B")
        D = A.shape[1]
        self._shard_ws(max(A.shape[0], B.shape[0]), 1, D, 0, 1)
        s = np.zeros(D, dtype=np.float64)
        self._check(self.lib.prohd_shift(self.h, A.data_ptr(), A.shape[0], B.data_ptr(), B.shape[0], D,
                                         s.ctypes.data))
        return s

    def local_moments(self, A_local, B_local, shift: np.ndarray) -> torch.Tensor:
        A, B = _as_points(A_local, "A"), _as_points(B_local, "B")
        D = A.shape[1]
        self._shard_ws(max(A.shape[0], B.shape[0]), 1, D, 0, 1)
        s = np.ascontiguousarray(shift, dtype=np.float64)
        out = torch.empty(2 * D + D * D, dtype=torch.float64, device=f"cuda:{self.device}")
        self._check(self.lib.prohd_local_moments(self.h, A.data_ptr() if A.numel() else None, A.shape[0],
                                                 B.data_ptr() if B.numel() else None, B.shape[0], D,
                                                 s.ctypes.data, out.data_ptr()))
        return out

    def local_colmax(self, A_local, B_local, shift: np.ndarray) -> torch.Tensor:
        """prohd_local_colmax: per-feature max |x - s| of this rank's rows (device fp32, D)."""
        A, B = _as_points(A_local, "A"), _as_points(B_local, "B")
        D = A.shape[1]
        self._shard_ws(max(A.shape[0], B.shape[0]), 1, D, 0, 1)
        s = np.ascontiguousarray(shift, dtype=np.float64)
        out = torch.empty(D, dtype=torch.float32, device=f"cuda:{self.device}")
        self._check(self.lib.prohd_local_colmax(self.h, A.data_ptr() if A.numel() else None, A.shape[0],
                                                B.data_ptr() if B.numel() else None, B.shape[0], D,
                                                s.ctypes.data, out.data_ptr()))
        return out

    def local_moments_i8(self, A_local, B_local, shift: np.ndarray, colmax: torch.Tensor) -> torch.Tensor:
        """prohd_local_moments_i8: [S_A | S_B | G] about s from the int8 Gram on the grid of the
        all-reduced column maxima `colmax` (device fp32, D)."""
        A, B = _as_points(A_local, "A"), _as_points(B_local, "B")
        D = A.shape[1]
        self._shard_ws(max(A.shape[0], B.shape[0]), 1, D, 0, 1)
        s = np.ascontiguousarray(shift, dtype=np.float64)
        cm = colmax.to(device=f"cuda:{self.device}", dtype=torch.float32).contiguous()
        out = torch.empty(2 * D + D * D, dtype=torch.float64, device=f"cuda:{self.device}")
        self._check(self.lib.prohd_local_moments_i8(self.h, A.data_ptr() if A.numel() else None, A.shape[0],
                                                    B.data_ptr() if B.numel() else None, B.shape[0], D,
                                                    s.ctypes.data, cm.data_ptr(), out.data_ptr()))
        return out

    def directions(self, moments: torch.Tensor, nA: int, nB: int, D: int, k: int, shift: np.ndarray):
        self._shard_ws(0, 1, D, k, 1)
        s = np.ascontiguousarray(shift, dtype=np.float64)
        dirs = torch.zeros(k + 1, D, dtype=torch.float64, device=f"cuda:{self.device}")
        nd = C.c_int32()
        self._check(self.lib.prohd_directions(self.h, moments.data_ptr(), nA, nB, D, k, s.ctypes.data,
                                              dirs.data_ptr(), C.byref(nd)))
        return dirs[: nd.value].contiguous(), int(nd.value)

    def local_candidates(self, X_local, row_offset: int, dirs: torch.Tensor, m: int):
        X = _as_points(X_local, "X")
        n_dirs, D = dirs.shape
        self._shard_ws(X.shape[0], 1, D, n_dirs - 1, m)
        val = torch.empty(n_dirs, 2, m, dtype=torch.float64, device=f"cuda:{self.device}")
        idx = torch.empty(n_dirs, 2, m, dtype=torch.int64, device=f"cuda:{self.device}")
        self._check(self.lib.prohd_local_candidates(self.h, X.data_ptr() if X.numel() else None, X.shape[0],
                                                    int(row_offset), D, dirs.data_ptr(), n_dirs, m,
                                                    val.data_ptr(), idx.data_ptr()))
        return val, idx

    def merge_union(self, vals: torch.Tensor, idxs: torch.Tensor, m: int, n_total: int) -> torch.Tensor:
        G, n_dirs = vals.shape[0], vals.shape[1]
        self._shard_ws(0, n_total, 1, n_dirs - 1, 1)
        cap = min(n_total, 2 * m * n_dirs)
        out = torch.empty(max(cap, 1), dtype=torch.int64, device=f"cuda:{self.device}")
        cnt = C.c_int64()
        self._check(self.lib.prohd_merge_union(self.h, vals.contiguous().data_ptr(), idxs.contiguous().data_ptr(),
                                               G, n_dirs, m, n_total, out.data_ptr(), C.byref(cnt)))
        return out[: cnt.value]

    def gather_owned(self, X_local, row_offset: int, union: torch.Tensor):
        X = _as_points(X_local, "X")
        D = X.shape[1]
        rows = torch.empty(max(union.numel(), 1), D, dtype=torch.float32, device=f"cuda:{self.device}")
        first, cnt = C.c_int64(), C.c_int64()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        self._check(self.lib.prohd_set_stream(self.h, C.c_void_p(stream)))
        self._check(self.lib.prohd_gather_owned(self.h, X.data_ptr() if X.numel() else None, X.shape[0],
                                                int(row_offset), D, union.data_ptr(), union.numel(),
                                                rows.data_ptr(), C.byref(first), C.byref(cnt)))
        return rows[: cnt.value], int(first.value), int(cnt.value)


_default: dict[int, Context] = {}


def set_option(name: str, value: int) -> None:
    """prohd_set_option: force a device variant (process-wide; value < 0 = default)."""
    lib = L.load()
    rc = lib.prohd_set_option(name.encode(), int(value))
    if rc != L.PROHD_OK:
        raise ProHDError(rc, f"unknown option {name!r}")


def get_option(name: str) -> int:
    lib = L.load()
    v = C.c_int64(0)
    rc = lib.prohd_get_option(name.encode(), C.byref(v))
    if rc != L.PROHD_OK:
        raise ProHDError(rc, f"unknown option {name!r}")
    return int(v.value)


class option:
    """Context manager: `with option("k6_split3", 1): ...` restores the previous value on exit."""

    def __init__(self, name: str, value: int):
        self.name, self.value, self.old = name, int(value), None

    def __enter__(self):
        self.old = get_option(self.name)
        set_option(self.name, self.value)
        return self

    def __exit__(self, *exc):
        set_option(self.name, self.old)
        return False


def context(device: int | None = None) -> Context:
    dev = torch.cuda.current_device() if device is None else int(device)
    if dev not in _default:
        _default[dev] = Context(dev)
    return _default[dev]


def directed_hd(A, B) -> dict:
    """h(A,B) = max_a min_b ||a-b|| with witness (Eq. (1))."""
    return context().directed_hd(A, B)


def hausdorff(A, B) -> dict:
    """H(A,B) = max(h(A,B), h(B,A)) (Eq. (1))."""
    return context().hausdorff(A, B)


def prohd_estimate(A, B, k: int, m: int, **kw) -> dict:
    """ProHD Alg. 3 estimate with k principal directions and m points per tail."""
    return context().prohd_estimate(A, B, k, m, **kw)


def unpack_key(key: int) -> tuple[float, int]:
    """(d2 as float32, global row) from a packed row-max key."""
    d2 = np.array([key >> 32], dtype=np.uint32).view(np.float32)[0]
    row = 0xFFFFFFFF - (key & 0xFFFFFFFF)
    return float(d2), int(row)
