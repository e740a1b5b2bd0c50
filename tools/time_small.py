"""Dev: wall-clock latency of one prohd_estimate call (device-resident inputs) at small configs,
and the library's kernel launches per call: python tools/time_small.py [cfg ...]"""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _opts  # noqa: E402
_opts.apply_env()
import torch
import datagen
from paper_2511_18207_b200 import Context

ctx = Context(0)
for cfg in [int(c) for c in (sys.argv[1:] or ["1", "2"])]:
    c = datagen.CONFIGS[cfg]
    A = torch.from_numpy(datagen.generate_set(cfg, "A")).cuda()
    B = torch.from_numpy(datagen.generate_set(cfg, "B")).cuda()
    for _ in range(3):
        r = ctx.prohd_estimate(A, B, c.k, c.m())
    l0 = ctx.launch_count()
    ts = []
    for _ in range(30):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = ctx.prohd_estimate(A, B, c.k, c.m())
        ts.append((time.perf_counter() - t0) * 1e3)
    nl = (ctx.launch_count() - l0) / 30
    ctx.enable_timing(True)
    r = ctx.prohd_estimate(A, B, c.k, c.m())
    tm = ctx.last_timings()
    ctx.enable_timing(False)
    print(f"cfg{cfg}: wall ms median {statistics.median(ts):.3f} min {min(ts):.3f}; launches/call {nl:.1f}; "
          f"phases {({k: round(v, 3) for k, v in tm.items() if k.endswith('_ms')})}; value {r['value']:.6f}", flush=True)
