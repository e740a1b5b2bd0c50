"""ncu target: one prohd_directions call per (D, k) on a prescribed spectrum."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2511_18207_b200 import Context
ctx = Context(0)
for D, k in [(4, 2), (64, 8), (256, 16)]:
    rng = np.random.default_rng(D)
    q, r = np.linalg.qr(rng.standard_normal((D, D)))
    lam = np.sort(rng.uniform(0.1, 10, D))[::-1]
    C = (q * lam) @ q.T
    mom = torch.from_numpy(np.concatenate([np.zeros(2 * D), (0.5 * (C + C.T) * 1000).ravel()])).cuda()
    ctx.directions(mom, 500, 500, D, k, np.zeros(D))
    torch.cuda.synchronize()
