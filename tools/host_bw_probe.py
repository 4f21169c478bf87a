"""Host memory write bandwidth into a pinned buffer with T threads (numpy
slice fills/copies release the GIL): decides whether expanding a compact
element store on the host can beat shipping the full store over PCIe.

    python tools/host_bw_probe.py
"""
import json
import os
import threading
import time

import numpy as np
import torch

N = 151 * 1024 * 1024 // 4  # the 2D-E-1M f32 store


def run(threads, dst, src):
    n = dst.size
    parts = [(i * n // threads, (i + 1) * n // threads) for i in range(threads)]

    def work(lo, hi):
        dst[lo:hi] = src[lo:hi]

    best = 1e9
    for _ in range(5):
        ts = [threading.Thread(target=work, args=p) for p in parts]
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        best = min(best, time.perf_counter() - t0)
    return dst.nbytes / best / 1e9


def main():
    dst = torch.empty(N, dtype=torch.float32).pin_memory().numpy()
    src = np.ones(N, dtype=np.float32)
    res = {"cores": os.cpu_count()}
    for t in (1, 2, 4, 8, 16, 32):
        if t <= 2 * (os.cpu_count() or 1):
            res[f"copy_GBs_{t}t"] = round(run(t, dst, src), 1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
