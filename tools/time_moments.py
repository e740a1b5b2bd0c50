"""Dev timing: the moments phase (K1) of prohd_estimate at one config, median of 7 (ms)."""
import os, sys, statistics
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
ts = []
for i in range(9):
    ctx.prohd_estimate(A, B, c.k, c.m())
    if i >= 2:
        ts.append(ctx.last_timings()["moments_ms"])
print(f"cfg{cfg} beta={os.environ.get('PROHD_OPT_K1_BETA_MILLI', '0')}: moments {statistics.median(ts):.3f} ms", flush=True)
