"""PCIe ceilings for the end-to-end path: pinned H2D / D2H copy bandwidth at
the e2e sizes of the default bench workload, next to the e2e call itself.

    python tools/pcie_probe.py [out.json]
"""
import json
import sys
import time
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1103_0066_b200 as fb  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def main():
    op, dim, ne, _ = bench.WORKLOADS["2d-elasticity-1m"]
    v, c, _ = bench.build_rank_mesh(op, dim, ne, 0, 1)
    var = fb.make_variant(op, dim, "f32", "strict")
    n = var.store_length(ne)
    out = {}
    dev = torch.empty(n, dtype=torch.float32, device="cuda")
    host = torch.empty(n, dtype=torch.float32).pin_memory()
    out["d2h_store_GBs"] = n * 4 / timed(lambda: host.copy_(dev, non_blocking=True)) * 1e-9
    hin = torch.empty(v.nbytes + c.nbytes, dtype=torch.uint8).pin_memory()
    din = torch.empty(hin.numel(), dtype=torch.uint8, device="cuda")
    out["h2d_mesh_GBs"] = hin.numel() / timed(lambda: din.copy_(hin, non_blocking=True)) * 1e-9
    out["d2h_store_ms"] = n * 4 / out["d2h_store_GBs"] * 1e-6
    hv, hc = torch.from_numpy(v).pin_memory().numpy(), torch.from_numpy(c).pin_memory().numpy()
    ho = host.numpy()
    out["e2e_ms"] = timed(lambda: fb.integrate_mesh(var, hv, hc, out=ho, devices=[0])) * 1e3
    print(json.dumps(out))
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
