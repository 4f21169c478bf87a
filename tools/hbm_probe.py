"""HBM ceilings for a store-dominated kernel: pure write, pure read, copy.

The roofline denominator in bench.py is the driver-measured copy bandwidth
(MEASURED_PEAKS.json).  Element integration is 64-98% stores, so the pure
write stream is measured here too and reported next to it.
"""
import json
import sys

import torch


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s = [torch.cuda.Event(enable_timing=True) for _ in range(reps)]
    e = [torch.cuda.Event(enable_timing=True) for _ in range(reps)]
    for i in range(reps):
        s[i].record()
        fn()
        e[i].record()
    torch.cuda.synchronize()
    return min(a.elapsed_time(b) for a, b in zip(s, e)) * 1e-3


def main():
    out = {}
    for mb in (160, 1024, 4096):
        n = mb << 20
        a = torch.empty(n // 4, dtype=torch.float32, device="cuda")
        b = torch.empty(n // 4, dtype=torch.float32, device="cuda")
        a.fill_(1.0)
        t = timed(lambda: b.fill_(3.0))
        out[f"write_{mb}MB_GBs"] = n / t * 1e-9
        t = timed(lambda: a.sum())
        out[f"read_{mb}MB_GBs"] = n / t * 1e-9
        t = timed(lambda: b.copy_(a))
        out[f"copy_{mb}MB_GBs"] = 2 * n / t * 1e-9
        del a, b
    print(json.dumps(out))
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
