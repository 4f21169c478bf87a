"""Quick kernel-only timing matrix (device-resident inputs, L2 flushed).

    python tools/kbench.py [--workloads a,b] [--modes strict,fast] [--precisions f32,f64] [--steps 10]

Prints one line per (workload, precision, mode): ms, GB/s, fraction of the
measured HBM copy bandwidth.  Development tool; bench.py is the contract.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1103_0066_b200 as fb  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--workloads", default="2d-elasticity-1m,3d-laplacian-16m,3d-elasticity-8m")
    p.add_argument("--modes", default="strict,fast")
    p.add_argument("--precisions", default="f32,f64")
    p.add_argument("--stores", default="auto")
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--elements", type=int, default=0, help="override elements per workload")
    a = p.parse_args()
    peak, _ = bench.peaks()
    scrub = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    scrub.fill_(1)
    st = torch.empty(2, dtype=torch.int64, device="cuda")
    sid = torch.cuda.current_stream().cuda_stream
    res = []
    for w in a.workloads.split(","):
        op, dim, ne, _ = bench.WORKLOADS[w]
        ne = a.elements or ne
        v, c, _ = bench.build_rank_mesh(op, dim, ne, 0, 1)
        nv_ref = int(np.unique(c).size)
        dv, dc = torch.from_numpy(v).cuda(), torch.from_numpy(c).cuda()
        for prec in a.precisions.split(","):
            for mode in a.modes.split(","):
                for store in a.stores.split(","):
                    var = fb.make_variant(op, dim, prec, mode, store=store)
                    out = torch.empty(var.store_length(ne), device="cuda",
                                      dtype=torch.float32 if prec == "f32" else torch.float64)
                    fb.status_reset(st, sid)
                    for _ in range(3):
                        fb.integrate_mesh_async(var, dv, dc, out, st, sid)
                    ms = []
                    for _ in range(a.steps):
                        scrub.view(torch.int64).sum()
                        torch.cuda._sleep(bench.GAP_CYCLES)
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record()
                        fb.integrate_mesh_async(var, dv, dc, out, st, sid)
                        e1.record()
                        torch.cuda.synchronize()
                        ms.append(e0.elapsed_time(e1))
                    fb.status_check(st, sid)
                    t = statistics.median(ms)
                    by = bench.algorithmic_bytes(op, dim, prec, c, nv_ref)
                    gbs = by / (t * 1e-3) * 1e-9
                    r = {"workload": w, "prec": prec, "mode": mode, "store": store, "ms": round(t, 4),
                         "GBs": round(gbs), "frac": round(gbs / peak, 3),
                         "Gelem_s": round(ne / (t * 1e-3) * 1e-9, 2)}
                    print(json.dumps(r), flush=True)
                    res.append(r)
    with open(os.path.join(ROOT, "gpurun_out", "kbench.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
