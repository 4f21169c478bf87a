"""Write profiles/ncu_traffic.json: per-launch DRAM traffic of the top kernel
(dram__bytes_read.sum + dram__bytes_write.sum from one `ncu --set full`
capture) keyed "workload:precision:mode", read by bench.py's roofline block.
Each entry records the hash of the kernel sources it was captured on
(bench.kernel_source_sha); bench.py reports traffic null once they change.

    python tools/ncu_traffic.py KEY report.ncu-rep [KEY report ...]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_traffic.json")
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def traffic(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, r = rows[0], rows[1], rows[2]
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(k)
        tot += float(r[i].replace(",", "")) * UNITS[u[i]]
    return tot


def main():
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    args = sys.argv[1:]
    sys.path.insert(0, ROOT)
    import bench

    sha = bench.kernel_source_sha()
    for key, rep in zip(args[::2], args[1::2]):
        data[key] = {"traffic": traffic(rep), "kernel_sha": sha, "report": os.path.basename(rep)}
        print(key, data[key])
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        json.dump(data, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
