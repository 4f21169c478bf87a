"""Pretty-print gpurun_out/ab.txt (tools/ab.sh output)."""
import json
import sys

for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab.txt"):
    if line.startswith("=="):
        print(line.strip())
        continue
    try:
        d = json.loads(line)
    except ValueError:
        print(line.rstrip())
        continue
    print(f"{d['workload']:18s} {d['prec']} {d['mode']:6s} {d['store']:7s} {d['ms']:8.4f} {d['frac']:.3f}")
