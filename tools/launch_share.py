"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, total device time and share of the captured time.

    python tools/launch_share.py gpurun_out/launches.csv
"""
import csv
import sys
from collections import defaultdict

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        agg[r[ki][:90]][0] += 1
        agg[r[ki][:90]][1] += float(r[vi].replace(",", "")) * SCALE[r[ui]]
    tot = sum(t for _, t in agg.values())
    print(f"{'launches':>8} {'total_us':>10} {'share':>6}  kernel")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n:8d} {t:10.1f} {100 * t / tot:5.1f}%  {k}")


if __name__ == "__main__":
    main()
