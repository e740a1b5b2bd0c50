"""Dev timing of K2 through prohd_directions on a prescribed spectrum; PROHD_OPT_EIG_STOP=1|2|3
stops after tridiagonalisation | bisection | inverse iteration (timing prefixes).
Optional arguments: D k (one case only)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _opts  # noqa: E402
_opts.apply_env()
import numpy as np
import torch
from paper_2511_18207_b200 import Context
ctx = Context(0)
ctx.enable_timing(True)
CASES = [(int(sys.argv[1]), int(sys.argv[2]))] if len(sys.argv) > 2 else [(64, 8), (128, 8), (256, 16), (256, 1)]
for D, k in CASES:
    rng = np.random.default_rng(D)
    q, r = np.linalg.qr(rng.standard_normal((D, D)))
    lam = np.sort(rng.uniform(0.1, 10, D))[::-1]
    C = (q * lam) @ q.T
    mom = torch.from_numpy(np.concatenate([np.zeros(2 * D), (0.5 * (C + C.T) * 1000).ravel()])).cuda()
    ts = []
    for _ in range(6):
        ctx.directions(mom, 500, 500, D, k, np.zeros(D))
        ts.append(ctx.last_timings()["eigen_ms"])
    print(f"D={D} k={k} stop={os.environ.get('PROHD_OPT_EIG_STOP', '0')}: eigen {statistics.median(ts[1:]):.3f} ms",
          flush=True)
