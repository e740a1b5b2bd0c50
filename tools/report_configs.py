"""Per-config report on one GPU: exact directed HD pairs/s, undirected HD
(fused bidirectional sweep) effective pairs/s, ProHD end-to-end ms with its phases, for all five
BASELINE configs at full size. Device-resident inputs, CUDA events, warm-up first.

    python tools/report_configs.py [cfg ...]   -> markdown table on stdout
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import datagen
from paper_2511_18207_b200 import Context


def timed(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    out = None
    for _ in range(reps):
        torch.cuda.synchronize()
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), out


def main():
    cfgs = [int(c) for c in sys.argv[1:]] or [1, 2, 3, 4, 5]
    ctx = Context(0)
    ctx.enable_timing(True)
    print("| cfg | n, D, k, m | directed h(A,B) ms | Gpair/s | undirected H ms | eff. Gpair/s | ProHD ms "
          "(moments / eigen / select / subset) | H | Ĥ | |I_A|, |I_B| |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for cfg in cfgs:
        c = datagen.CONFIGS[cfg]
        A = torch.from_numpy(datagen.generate_set(cfg, "A")).cuda()
        B = torch.from_numpy(datagen.generate_set(cfg, "B")).cuda()
        n = A.shape[0]
        reps = 1 if n >= 1_000_000 else 3
        ctx.directed_hd(A, B)  # warm-up (workspace, descriptors)
        t_dir, _ = timed(lambda: ctx.directed_hd(A, B), reps)
        ctx.hausdorff(A, B)
        t_und, h = timed(lambda: ctx.hausdorff(A, B), reps)
        ctx.prohd_estimate(A, B, c.k, c.m())
        runs = []
        for _ in range(5):
            e = ctx.prohd_estimate(A, B, c.k, c.m())
            runs.append(ctx.last_timings())
        med = {k: statistics.median(t[k] for t in runs) for k in
               ("moments_ms", "eigen_ms", "select_ms", "subset_ms", "total_ms")}
        pairs = float(n) * float(B.shape[0])
        print(f"| {cfg} | {n}, {A.shape[1]}, {c.k}, {c.m()} | {t_dir:.2f} | {pairs / t_dir / 1e6:.1f} | "
              f"{t_und:.2f} | {2 * pairs / t_und / 1e6:.1f} | **{med['total_ms']:.2f}** ({med['moments_ms']:.2f} / "
              f"{med['eigen_ms']:.2f} / {med['select_ms']:.2f} / {med['subset_ms']:.2f}) | {h['value']:.6g} | "
              f"{e['value']:.6g} | {e['size_a']}, {e['size_b']} |", flush=True)
        del A, B
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
