"""Dev timing: the fused bidirectional sweep (hausdorff) on the single-block K6 (default) against the
CTA-pair K6 (option k6_bidir_2a = 2), interleaved in one process; kernel time from the library's events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_18207_b200 import Context, option
ctx = Context(0)
shapes = [(65536, 262144, 256), (65536, 262144, 128), (13352, 13233, 256), (32311, 32121, 256), (17962, 17972, 128)]
for (nA, nB, D) in shapes:
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(nA, D, device="cuda", generator=g)
    B = torch.randn(nB, D, device="cuda", generator=g)
    reps = 3 if nA * nB > 1e9 else 20
    for rnd in range(2):
        for v in (0, 2):
            with option("k6_bidir_2a", v):
                h = ctx.hausdorff(A, B)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    h = ctx.hausdorff(A, B)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / reps
            print(f"nA={nA} nB={nB} D={D} bidir_2a={v}: {ms:.3f} ms/call  {2.0 * nA * nB / ms / 1e6:.0f} eff Gpair/s  "
                  f"H={h['value']:.6f}", flush=True)
