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
    a = p.parse_args()
    op, dim, ne, _ = bench.WORKLOADS[a.workload]
    v, c, _ = bench.build_rank_mesh(op, dim, ne, 0, 1)
    var = fb.make_variant(op, dim, a.precision, a.mode, element_batch_size=128, store=a.store)
    dv, dc = torch.from_numpy(v).cuda(), torch.from_numpy(c).cuda()
    out = torch.empty(var.store_length(ne), dtype=torch.float32 if a.precision == "f32" else torch.float64,
                      device="cuda")
    st = torch.empty(2, dtype=torch.int64, device="cuda")
    sid = torch.cuda.current_stream().cuda_stream
    fb.status_reset(st, sid)
    for _ in range(a.reps):
        fb.integrate_mesh_async(var, dv, dc, out, st, sid)
    fb.status_check(st, sid)
    torch.cuda.synchronize()
    print("ok", a)


if __name__ == "__main__":
    main()
