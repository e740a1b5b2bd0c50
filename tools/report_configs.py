"""Per-config report on one GPU: exact directed HD pairs/s, undirected HD
(fused bidirectional sweep) effective pairs/s, ProHD end-to-end ms with its phases, and each phase's
roofline fraction, for all five BASELINE configs at full size. Device-resident inputs, CUDA events
inside the library, warm-up first.

    python tools/report_configs.py [--json out.json] [cfg ...]   -> markdown table on stdout
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
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
    args = sys.argv[1:]
    jpath = None
    if "--json" in args:
        i = args.index("--json")
        jpath = args[i + 1]
        del args[i:i + 2]
    cfgs = [int(c) for c in args] or [1, 2, 3, 4, 5]
    ctx = Context(0)
    ctx.enable_timing(True)
    pk = bench.peaks()
    rows = []
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
        t_dir, d = timed(lambda: ctx.directed_hd(A, B), reps)
        k6 = ctx.last_timings()
        ctx.hausdorff(A, B)
        t_und, h = timed(lambda: ctx.hausdorff(A, B), reps)
        ctx.prohd_estimate(A, B, c.k, c.m())
        runs = []
        for _ in range(5):
            e = ctx.prohd_estimate(A, B, c.k, c.m())
            runs.append(ctx.last_timings())
        med = {k: statistics.median(t[k] for t in runs) for k in
               ("moments_ms", "eigen_ms", "select_ms", "subset_ms", "total_ms", "prep_ms")}
        pairs = float(n) * float(B.shape[0])
        D = A.shape[1]
        k6_tf = 6.0 * D * pairs / (k6["dist_ms"] / 1e3) / 1e12
        rec = {"cfg": cfg, "n": n, "D": D, "k": c.k, "m": c.m(),
               "exact": {"directed_ms": t_dir, "directed_Gpair_s": pairs / t_dir / 1e6,
                         "undirected_ms": t_und, "undirected_eff_Gpair_s": 2 * pairs / t_und / 1e6,
                         "k6_ms": k6["dist_ms"], "k6_tflops_fp16": k6_tf,
                         "k6_frac_fp16_burst": k6_tf / pk["bf16_tflops"], "H": h["value"], "h_ab": d["dist"]},
               "prohd": {"ms": med["total_ms"], "phases_ms": med, "value": e["value"], "size_a": e["size_a"],
                         "size_b": e["size_b"],
                         "kernels": bench.phase_rooflines(c, runs[-1], k6, e, pk)}}
        rows.append(rec)
        print(f"| {cfg} | {n}, {D}, {c.k}, {c.m()} | {t_dir:.2f} | {pairs / t_dir / 1e6:.1f} | "
              f"{t_und:.2f} | {2 * pairs / t_und / 1e6:.1f} | **{med['total_ms']:.2f}** ({med['moments_ms']:.2f} / "
              f"{med['eigen_ms']:.2f} / {med['select_ms']:.2f} / {med['subset_ms']:.2f}) | {h['value']:.6g} | "
              f"{e['value']:.6g} | {e['size_a']}, {e['size_b']} |", flush=True)
        del A, B
        torch.cuda.empty_cache()
    if jpath:
        with open(jpath, "w") as f:
            json.dump({"gpu": torch.cuda.get_device_name(0), "peaks": pk, "configs": rows}, f, indent=1)


if __name__ == "__main__":
    main()
