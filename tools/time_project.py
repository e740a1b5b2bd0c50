"""Dev timing: K3 alone through the prohd_project hook, 2M x 256 points, 17 directions (cfg5 shape)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _opts  # noqa: E402
_opts.apply_env()
import numpy as np
import torch
from paper_2511_18207_b200 import Context
n, D, L = 2_000_000, 256, 17
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn((n, D), device="cuda", generator=g)
U = np.linalg.qr(np.random.default_rng(0).standard_normal((D, L)))[0].T.copy()
ctx = Context(0)
for _ in range(3):
    ctx.project(X, U)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(10):
    e0.record(); ctx.project(X, U); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
t = sorted(ts)[len(ts) // 2]
print(f"dbg={os.environ.get('PROHD_OPT_K3_DBG', '0')} simt={os.environ.get('PROHD_OPT_K3_SIMT', '0')}: {t:.3f} ms "
      f"(call incl. U conversion + readback), {n * D * 4 / t / 1e6:.0f} GB/s", flush=True)
