"""Launch the fused integration kernel a few times on one workload (for ncu).

    python tools/run_kernel.py --workload 2d-elasticity-1m --precision f32 [--mode strict] [--reps 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1103_0066_b200 as fb  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--workload", default="2d-elasticity-1m")
    p.add_argument("--precision", default="f32")
    p.add_argument("--mode", default="strict")
    p.add_argument("--store", default="auto")
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--elements", type=int, default=0, help="override the workload's element count")
    p.add_argument("--op", default="", help="override the workload's operator")
    a = p.parse_args()
    op, dim, ne, _ = bench.WORKLOADS[a.workload]
    op = a.op or op
    ne = a.elements or ne
    from paper_1103_0066_b200 import mesh_prefix
    v, c, _ = mesh_prefix(dim, ne, 0.15 if ne <= (1 << 24) else 0.0, 42)
    w = None
    if op == "weighted-laplacian":
        import numpy as np
        w = torch.from_numpy(np.ascontiguousarray(1.0 + v.reshape(-1, dim)[c.reshape(-1, dim + 1), 0].ravel())).cuda()
    var = fb.make_variant(op, dim, a.precision, a.mode, element_batch_size=128, store=a.store)
    dv, dc = torch.from_numpy(v).cuda(), torch.from_numpy(c).cuda()
    out = torch.empty(var.store_length(ne), dtype=torch.float32 if a.precision == "f32" else torch.float64,
                      device="cuda")
    st = torch.empty(2, dtype=torch.int64, device="cuda")
    sid = torch.cuda.current_stream().cuda_stream
    fb.status_reset(st, sid)
    for _ in range(a.reps):
        fb.integrate_mesh_async(var, dv, dc, out, st, sid, coefficients=w)
    fb.status_check(st, sid)
    torch.cuda.synchronize()
    print("ok", a)


if __name__ == "__main__":
    main()
