"""Probe K6's split-product arithmetic on adversarial constant rows (dev tool).

For each x in a list of fp32 values and each D: A = {x.1}, B = {x.1, -x.1} (centre 0), the GPU row
minimum of the single row is the computed d^2 of the self pair (exact value 0), printed relative to
the Q17 budget scale 2 D x^2. Variants: default split, k6_split3 (literal 3xTF32), k6_variant 1/3."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np
import torch
from paper_2511_18207_b200 import Context, option

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_exact import _fp16_split_rel_err as _split_product_rel_err  # noqa: E402

ctx = Context(0)
m = np.arange(1 << 23, dtype=np.uint32)
xs = (m | np.uint32(127 << 23)).view(np.float32)
err = _split_product_rel_err(xs)
o = np.argsort(-np.abs(err))
rng = np.random.default_rng(0)
vals = np.concatenate([xs[o[:16]], xs[rng.integers(0, 1 << 23, 48)]]).astype(np.float32)
emu = _split_product_rel_err(vals)


def run(D, variant=None, split3=None):
    out = []
    for x in vals:
        A = torch.full((1, D), float(x), dtype=torch.float32, device="cuda")
        B = torch.cat([A, -A])
        r = ctx.directed_hd_rowmin(A, B).cpu().numpy()[0]
        out.append(float(r) / (2 * D * float(x) ** 2))
    return np.array(out)


for D in (8, 16, 64, 256):
    for name, opts in (("default", {}), ("split3", {"k6_split3": 1}), ("v1", {"k6_variant": 1}),
                       ("v3", {"k6_variant": 3}), ("v1split3", {"k6_variant": 1, "k6_split3": 1})):
        cms = [option(k, v) for k, v in opts.items()]
        for c in cms:
            c.__enter__()
        r = run(D)
        for c in cms[::-1]:
            c.__exit__()
        print(f"D={D:4d} {name:8s} max rel {r.max():.3e} at x={vals[r.argmax()]!r} (emu {-emu[r.argmax()]:.2e}); "
              f"mean {r.mean():.2e}; worst16 mean {r[:16].mean():.2e}, random48 mean {r[16:].mean():.2e}", flush=True)
    if D == 256:
        for i in range(16):
            print(f"   x={vals[i]!r} emu {-emu[i]:.3e}", flush=True)
