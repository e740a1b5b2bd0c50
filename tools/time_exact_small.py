"""Dev: wall-clock latency of directed_hd / hausdorff at the small configs (device inputs), graph
replay (default) and eager (option graph = 0): python tools/time_exact_small.py [cfg ...]"""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import datagen
from paper_2511_18207_b200 import Context, option

ctx = Context(0)
for cfg in [int(c) for c in (sys.argv[1:] or ["1", "2"])]:
    A = torch.from_numpy(datagen.generate_set(cfg, "A")).cuda()
    B = torch.from_numpy(datagen.generate_set(cfg, "B")).cuda()
    for g in (-1, 0):
        with option("graph", g):
            out = {}
            for name, fn in (("directed", ctx.directed_hd), ("hausdorff", ctx.hausdorff)):
                for _ in range(3):
                    fn(A, B)
                ts = []
                for _ in range(20):
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    fn(A, B)
                    ts.append((time.perf_counter() - t0) * 1e3)
                out[name] = statistics.median(ts)
        print(f"cfg{cfg} {'graph' if g else 'eager'}: directed {out['directed']:.3f} ms, hausdorff {out['hausdorff']:.3f} ms",
              flush=True)
