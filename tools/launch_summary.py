"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list as a markdown table."""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
        except ValueError:
            continue
        name = r[ki].replace("(anonymous namespace)::", "").split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print("| kernel | launches | total ms | share |")
    print("|---|---|---|---|")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {c} | {v:.3f} | {100 * v / tot:.2f}% |")


if __name__ == "__main__":
    main()
