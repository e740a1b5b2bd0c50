"""ctypes declarations for libprohd.so (include/prohd.h). Argument marshalling only."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libprohd.so")

PROHD_OK = 0
PROHD_E_INVALID = 2
PROHD_E_DATA = 3
PROHD_E_INTERNAL = 4
PROHD_E_CUDA = 5
PROHD_E_WORKSPACE = 6
PROHD_E_NOTIMPL = 7
PROHD_E_DEVICE = 8
PROHD_WS_HOST_INPUTS = 1
PROHD_WS_CERTIFIED = 2

STATUS_NAMES = {0: "PROHD_OK", 2: "PROHD_E_INVALID", 3: "PROHD_E_DATA", 4: "PROHD_E_INTERNAL",
                5: "PROHD_E_CUDA", 6: "PROHD_E_WORKSPACE", 7: "PROHD_E_NOTIMPL", 8: "PROHD_E_DEVICE"}

# every symbol include/prohd.h declares (checked by tests/test_abi.py)
EXPORTED = [
    "prohd_create", "prohd_destroy", "prohd_set_stream", "prohd_last_error", "prohd_version",
    "prohd_launch_count",
    "prohd_set_option",
    "prohd_get_option",
    "prohd_workspace_bytes", "prohd_set_workspace", "directed_hd", "hausdorff", "directed_hd_rowmin", "hausdorff_minima", "prohd_covariance",
    "prohd_estimate", "prohd_estimate_certified", "prohd_estimate_alpha", "hausdorff_subsets",
    "prohd_estimate_with_dirs", "prohd_bounds", "directed_hd_local", "prohd_centre", "directed_hd_witness",
    "prohd_project",
    "prohd_enable_timing", "prohd_last_timings",
    "prohd_shard_workspace_bytes", "prohd_shift", "prohd_local_moments", "prohd_local_colmax",
    "prohd_local_moments_i8", "prohd_directions",
    "prohd_local_candidates", "prohd_merge_union", "prohd_gather_owned",
]


class Directed(C.Structure):
    _fields_ = [("dist", C.c_double), ("dist2", C.c_double), ("a", C.c_int64), ("b", C.c_int64),
                ("dist2_tc", C.c_double)]


class HD(C.Structure):
    _fields_ = [("value", C.c_double), ("ab", Directed), ("ba", Directed)]


class Est(C.Structure):
    _fields_ = [("value", C.c_double), ("ab", Directed), ("ba", Directed), ("size_a", C.c_int64),
                ("size_b", C.c_int64), ("n_dirs", C.c_int32), ("_pad", C.c_int32)]


class Timings(C.Structure):
    _fields_ = [("total_ms", C.c_double), ("h2d_ms", C.c_double), ("prep_ms", C.c_double),
                ("dist_ms", C.c_double), ("reduce_ms", C.c_double), ("moments_ms", C.c_double),
                ("eigen_ms", C.c_double), ("select_ms", C.c_double), ("subset_ms", C.c_double),
                ("dist_launches", C.c_int32), ("kernel_launches", C.c_int32)]


_lib = None


def load() -> C.CDLL:
    """Load libprohd.so; raises (never falls back) if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not found: build it with `python -m paper_2511_18207_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    vp, i64, i32, f = C.c_void_p, C.c_int64, C.c_int32, C.c_int
    lib.prohd_create.argtypes = [f, vp, C.POINTER(vp)]
    lib.prohd_destroy.argtypes = [vp]
    lib.prohd_set_stream.argtypes = [vp, vp]
    lib.prohd_last_error.argtypes = [vp]
    lib.prohd_last_error.restype = C.c_char_p
    lib.prohd_version.restype = C.c_char_p
    lib.prohd_launch_count.argtypes = [C.POINTER(C.c_int64)]
    lib.prohd_set_option.argtypes = [C.c_char_p, i64]
    lib.prohd_get_option.argtypes = [C.c_char_p, C.POINTER(C.c_int64)]
    lib.prohd_workspace_bytes.argtypes = [i64, i64, i32, i32, i64, C.c_uint32]
    lib.prohd_workspace_bytes.restype = C.c_size_t
    lib.prohd_set_workspace.argtypes = [vp, vp, C.c_size_t]
    lib.directed_hd.argtypes = [vp, vp, i64, vp, i64, i32, C.POINTER(Directed)]
    lib.hausdorff.argtypes = [vp, vp, i64, vp, i64, i32, C.POINTER(HD)]
    lib.hausdorff_minima.argtypes = [vp, vp, i64, vp, i64, i32, vp, vp, C.POINTER(HD)]
    lib.prohd_covariance.argtypes = [vp, vp, i64, vp, i64, i32, vp, vp, C.POINTER(C.c_int32)]
    lib.directed_hd_rowmin.argtypes = [vp, vp, i64, vp, i64, i32, vp]
    lib.prohd_estimate.argtypes = [vp, vp, i64, vp, i64, i32, i32, i64, C.POINTER(Est), vp, vp, vp]
    lib.prohd_estimate_certified.argtypes = [vp, vp, i64, vp, i64, i32, i32, i64, C.POINTER(Est), vp, vp, vp]
    lib.prohd_estimate_alpha.argtypes = [vp, vp, i64, vp, i64, i32, C.c_double, C.POINTER(Est), vp, vp, vp]
    lib.hausdorff_subsets.argtypes = [vp, vp, i64, vp, i64, vp, i64, vp, i64, i32, C.POINTER(HD)]
    lib.prohd_bounds.argtypes = [vp, vp, i64, vp, i64, i32, vp, i32, vp, vp]
    lib.prohd_estimate_with_dirs.argtypes = [vp, vp, i64, vp, i64, i32, i32, i64, vp, C.POINTER(Est), vp, vp]
    lib.directed_hd_local.argtypes = [vp, vp, i64, i64, vp, i64, i32, vp, C.POINTER(C.c_uint64)]
    lib.prohd_centre.argtypes = [vp, vp, i64, vp, i64, i32, vp]
    lib.prohd_project.argtypes = [vp, vp, i64, i32, vp, i32, vp, vp]
    lib.directed_hd_witness.argtypes = [vp, vp, vp, i64, i32, C.POINTER(Directed)]
    lib.prohd_enable_timing.argtypes = [vp, f]
    lib.prohd_shard_workspace_bytes.argtypes = [i64, i64, i32, i32, i64, C.c_uint32]
    lib.prohd_shard_workspace_bytes.restype = C.c_size_t
    lib.prohd_shift.argtypes = [vp, vp, i64, vp, i64, i32, vp]
    lib.prohd_local_moments.argtypes = [vp, vp, i64, vp, i64, i32, vp, vp]
    lib.prohd_local_colmax.argtypes = [vp, vp, i64, vp, i64, i32, vp, vp]
    lib.prohd_local_moments_i8.argtypes = [vp, vp, i64, vp, i64, i32, vp, vp, vp]
    lib.prohd_directions.argtypes = [vp, vp, i64, i64, i32, i32, vp, vp, C.POINTER(C.c_int32)]
    lib.prohd_local_candidates.argtypes = [vp, vp, i64, i64, i32, vp, i32, i64, vp, vp]
    lib.prohd_merge_union.argtypes = [vp, vp, vp, i32, i32, i64, i64, vp, C.POINTER(C.c_int64)]
    lib.prohd_gather_owned.argtypes = [vp, vp, i64, i64, i32, vp, i64, vp, C.POINTER(C.c_int64),
                                       C.POINTER(C.c_int64)]
    lib.prohd_last_timings.argtypes = [vp, C.POINTER(Timings)]
    for name in EXPORTED:
        fn = getattr(lib, name)
        if name not in ("prohd_last_error", "prohd_version", "prohd_workspace_bytes",
                        "prohd_shard_workspace_bytes"):
            fn.restype = C.c_int
    _lib = lib
    return lib
