"""Dev check: GPU directions vs the fp64 oracle's at a config's full size (angles, C residuals,
selection equality). Run with PROHD_OPT_SHIFT=0/1 to compare the Gram paths."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _opts  # noqa: E402
_opts.apply_env()
import numpy as np
import torch
import datagen
from oracle import prohd as OP
from paper_2511_18207_b200 import Context
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = datagen.CONFIGS[cfg]
A = datagen.generate_set(cfg, "A"); B = datagen.generate_set(cfg, "B")
ctx = Context(0)
g = ctx.prohd_estimate(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), c.k, c.m(), return_dirs=True,
                       return_indices=True)
ref = OP.estimate(A, B, c.k, c.m())
U, R, C = g["U"], ref["U"], ref["C"]
cn = np.linalg.norm(C, 2)
ang = [float(np.linalg.norm(U[:, l] - (U[:, l] @ R[:, l]) * R[:, l])) for l in range(U.shape[1])]
res = [float(np.linalg.norm(C @ U[:, l] - (U[:, l] @ C @ U[:, l]) * U[:, l]) / cn) for l in range(1, U.shape[1])]
print(f"cfg{cfg} shift={os.environ.get('PROHD_OPT_SHIFT', 'auto')}: max sin-angle {max(ang):.3e}, max residual/||C|| "
      f"{max(res):.3e}, sets equal {np.array_equal(g['IA'], ref['IA']) and np.array_equal(g['IB'], ref['IB'])}, "
      f"H^ {g['value']:.9f} vs {ref['value']:.9f}", flush=True)
