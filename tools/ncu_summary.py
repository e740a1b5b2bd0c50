"""Summarise an `ncu --page raw --csv` export as a markdown table (one row per launch).

    python tools/ncu_summary.py gpurun_out/<tag>_raw.csv [kernel-substring ...]
"""
import csv
import sys

COLS = [
    ("ms", "gpu__time_duration.sum", 1.0),
    ("DRAM rd GB", "dram__bytes_read.sum", None),
    ("DRAM wr GB", "dram__bytes_write.sum", None),
    ("DRAM %", "dram__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("SM %", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("tensor %", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("DMMA % act", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    ("fp64 % act", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    ("SM GHz", "sm__cycles_elapsed.avg.per_second", 1.0),
]
UNIT = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3,
        "ms": 1.0, "us": 1e-3, "ns": 1e-6, "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6,
        "Ghz": 1.0, "Mhz": 1e-3, "hz": 1e-9, "cycle/second": 1e-9, "cycle/nsecond": 1.0, "%": 1.0}


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    h, units = rows[0], rows[1]
    filt = sys.argv[2:]
    idx = {c: i for i, c in enumerate(h)}
    print("| kernel | grid | block | " + " | ".join(c[0] for c in COLS) + " |")
    print("|---" * (3 + len(COLS)) + "|")
    for r in rows[2:]:
        name = r[idx["Kernel Name"]]
        if filt and not any(f in name for f in filt):
            continue
        cells = []
        for _, col, _ in COLS:
            i = idx.get(col)
            if i is None or not r[i]:
                cells.append("-")
                continue
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                cells.append(r[i])
                continue
            v *= UNIT.get(units[i], 1.0)
            cells.append(f"{v:.3f}" if abs(v) < 100 else f"{v:.1f}")
        short = name.replace("(anonymous namespace)::", "").split("(")[0][:48]
        print(f"| `{short}` | {r[idx['Grid Size']]} | {r[idx['Block Size']]} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main()
