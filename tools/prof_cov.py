"""Dev: time / profile step 1a (prohd_covariance) at a BASELINE config: python tools/prof_cov.py [cfg] [reps]"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _opts  # noqa: E402
_opts.apply_env()
import torch
import datagen
from paper_2511_18207_b200 import Context

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
A = torch.from_numpy(datagen.generate_set(cfg, "A")).cuda()
B = torch.from_numpy(datagen.generate_set(cfg, "B")).cuda()
ctx = Context(0)
ctx.enable_timing(True)
ts = []
for _ in range(reps):
    mu, C, path = ctx.covariance(A, B)
    ts.append(ctx.last_timings()["moments_ms"])
print(f"cfg{cfg} path={'int8' if path else 'dmma'} moments ms: {[round(t, 3) for t in ts]} median {statistics.median(ts):.3f}",
      flush=True)
