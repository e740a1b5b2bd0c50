"""Dev probe: the CTA-pair K6 (option k6_variant = 2) below its default range (D < 128): row minima against the
single-block kernel (bitwise) and interleaved timing of 65536 x 262144 directed sweeps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_18207_b200 import Context, option
ctx = Context(0)
for (nA, nB, D) in [(700, 2000, 16), (513, 1100, 40), (2000, 2500, 64), (257, 4099, 96), (20000, 3001, 100)]:
    g = torch.Generator(device="cuda").manual_seed(D)
    A = torch.randn(nA, D, device="cuda", generator=g)
    B = torch.randn(nB, D, device="cuda", generator=g) * 1.3 + 0.2
    with option("k6_variant", 1):
        r1 = ctx.directed_hd_rowmin(A, B)
    with option("k6_variant", 2):
        r2 = ctx.directed_hd_rowmin(A, B)
    print(f"parity nA={nA} nB={nB} D={D}: bitwise equal {bool(torch.equal(r1, r2))}  max abs diff {float((r1 - r2).abs().max()):.3e}", flush=True)
nA, nB = 65536, 262144
for D in (32, 64, 96):
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(nA, D, device="cuda", generator=g)
    B = torch.randn(nB, D, device="cuda", generator=g)
    for rnd in range(2):
        for v in (1, 2):
            with option("k6_variant", v):
                ctx.directed_hd(A, B)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(40):
                    ctx.directed_hd(A, B)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 40
            print(f"D={D} k6_variant={v}: {ms:.3f} ms/call  {nA * nB / ms / 1e6:.0f} Gpair/s", flush=True)
