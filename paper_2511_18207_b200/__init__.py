"""B200-native ProHD hot path (arxiv 2511.18207): exact and projection-guided
Hausdorff distance on sm_100a tensor cores, behind the C ABI in include/prohd.h.

The compute lives in libprohd.so (paper_2511_18207_b200/csrc); this package is
the thin Python binding (argument marshalling) plus the multi-GPU driver.
"""
from .api import (Context, ProHDError, context, directed_hd, get_option, hausdorff,  # noqa: F401
                  option, prohd_estimate, set_option, unpack_key)

__version__ = "0.1.0"
