"""Dev timing: directed exact HD throughput (Gpair/s) on synthetic N(0,1) data."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _opts  # noqa: E402
_opts.apply_env()
import time

import torch

from paper_2511_18207_b200 import Context

ctx = Context(0)
for (nA, nB, D) in [(16384, 65536, 256), (65536, 262144, 256), (65536, 262144, 128), (65536, 262144, 64),
                    (65536, 262144, 16)]:
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(nA, D, device="cuda", generator=g)
    B = torch.randn(nB, D, device="cuda", generator=g)
    ctx.directed_hd(A, B)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    ev0.record()
    for _ in range(reps):
        r = ctx.directed_hd(A, B)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / reps
    gp = nA * nB / ms / 1e6
    print(f"nA={nA} nB={nB} D={D}: {ms:.2f} ms  {gp:.1f} Gpair/s  {gp*6*D/1e3:.1f} executed-TFLOP/s  d={r['dist']:.4f}",
          flush=True)
