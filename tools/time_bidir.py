"""Dev timing: hausdorff() (one fused bidirectional sweep) vs two directed_hd calls."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _opts  # noqa: E402
_opts.apply_env()
import torch
from paper_2511_18207_b200 import Context
ctx = Context(0)
for (nA, nB, D) in [(65536, 262144, 256), (65536, 262144, 64), (262144, 262144, 16)]:
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(nA, D, device="cuda", generator=g)
    B = torch.randn(nB, D, device="cuda", generator=g)
    ctx.hausdorff(A, B); ctx.directed_hd(A, B)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(); h = ctx.hausdorff(A, B); e[1].record(); d1 = ctx.directed_hd(A, B); d2 = ctx.directed_hd(B, A); e[2].record()
    torch.cuda.synchronize()
    t_h, t_2 = e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])
    print(f"nA={nA} nB={nB} D={D}: hausdorff {t_h:.2f} ms ({2*nA*nB/t_h/1e6:.0f} eff Gpair/s), 2x directed {t_2:.2f} ms; "
          f"H={h['value']:.5f} vs {max(d1['dist'], d2['dist']):.5f}", flush=True)
