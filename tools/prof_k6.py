"""ncu target: one full-machine K6 launch (37888 x 262144, D=256) via directed_hd."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _opts  # noqa: E402
_opts.apply_env()
import torch
from paper_2511_18207_b200 import Context
ctx = Context(0)
g = torch.Generator(device="cuda").manual_seed(0)
nA, nB, D = 37888, 262144, int(sys.argv[1]) if len(sys.argv) > 1 else 256
A = torch.randn(nA, D, device="cuda", generator=g)
B = torch.randn(nB, D, device="cuda", generator=g)
bidir = len(sys.argv) > 2 and sys.argv[2] == "bidir"  # the fused bidirectional sweep (hausdorff)
r = ctx.hausdorff(A, B) if bidir else ctx.directed_hd(A, B)
print(nA, nB, D, r["value"] if bidir else r["dist"])
