"""Dev timing: prohd_estimate phases (in-library CUDA events) per config, median of 5 runs."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _opts  # noqa: E402
_opts.apply_env()
import torch
import datagen
from paper_2511_18207_b200 import Context
ctx = Context(0)
ctx.enable_timing(True)
for cfg in [int(c) for c in (sys.argv[1:] or ["5", "4", "3", "2"])]:
    c = datagen.CONFIGS[cfg]
    A = torch.from_numpy(datagen.generate_set(cfg, "A")).cuda()
    B = torch.from_numpy(datagen.generate_set(cfg, "B")).cuda()
    runs = []
    for _ in range(6):
        r = ctx.prohd_estimate(A, B, c.k, c.m())
        runs.append(ctx.last_timings())
    runs = runs[1:]
    keys = ("moments_ms", "eigen_ms", "select_ms", "subset_ms", "total_ms")
    med = {k: statistics.median(t[k] for t in runs) for k in keys}
    print(f"cfg{cfg}: " + " ".join(f"{k[:-3]}={v:.3f}" for k, v in med.items()) +
          f"  value={r['value']:.6f} |I|={r['size_a']},{r['size_b']}", flush=True)
    del A, B
    torch.cuda.empty_cache()
