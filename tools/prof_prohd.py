"""ncu target: one prohd_estimate at cfg5 (n=2M, D=256, k=16, m=1000)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _opts  # noqa: E402
_opts.apply_env()
import torch
import datagen
from paper_2511_18207_b200 import Context
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
c = datagen.CONFIGS[cfg]
A = torch.from_numpy(datagen.generate_set(cfg, "A")).cuda()
B = torch.from_numpy(datagen.generate_set(cfg, "B")).cuda()
ctx = Context(0)
ctx.enable_timing(True)
r = ctx.prohd_estimate(A, B, c.k, c.m())
print(r["value"], ctx.last_timings())
