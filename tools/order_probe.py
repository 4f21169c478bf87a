"""Assembly kernel time with and without the Morton group schedule
(AssemblyPlan.order_groups) on the benchmark mesh and on the same mesh with
its vertices renumbered at random (a badly ordered mesh).

    python tools/order_probe.py [--workload 3d-elasticity-8m] [--prec f32]
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


def timed(fn, steps, scrub, stream):
    for _ in range(3):
        fn()
    ms = []
    for _ in range(steps):
        scrub.view(torch.int64).sum()
        torch.cuda._sleep(bench.GAP_CYCLES)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return statistics.median(ms)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--workload", default="3d-elasticity-8m")
    p.add_argument("--prec", default="f32")
    p.add_argument("--steps", type=int, default=10)
    a = p.parse_args()
    op, dim, ne, _ = bench.WORKLOADS[a.workload]
    v, c, _ = bench.build_rank_mesh(op, dim, ne, 0, 1)
    nv = v.size // dim
    scrub = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    scrub.fill_(1)
    stream = torch.cuda.current_stream()
    sid = stream.cuda_stream
    perm = np.random.default_rng(1).permutation(nv).astype(np.int32)  # old id -> new id
    vp = np.empty_like(v.reshape(-1, dim))
    vp[perm] = v.reshape(-1, dim)
    meshes = {"benchmark": (v, c), "renumbered": (np.ascontiguousarray(vp.ravel()), perm[c])}
    st = torch.empty(2, dtype=torch.int64, device="cuda")
    for name, (vv, cc) in meshes.items():
        dv, dc = torch.from_numpy(vv).cuda(), torch.from_numpy(np.ascontiguousarray(cc)).cuda()
        var = fb.make_variant(op, dim, a.prec, "strict")
        store = torch.empty(var.store_length(ne), device="cuda",
                            dtype=torch.float32 if a.prec == "f32" else torch.float64)
        fb.status_reset(st, sid)
        fb.integrate_mesh_async(var, dv, dc, store, st, sid)
        fb.status_check(st, sid)
        g = fb.pack_geometry(dv, dc, dim, 128, a.prec)
        plan = fb.AssemblyPlan(op, dim, dc, nv)
        vals = torch.empty(plan.nnz, device="cuda", dtype=store.dtype)
        row = {"mesh": name, "workload": a.workload, "prec": a.prec}
        for order in (False, True):
            plan.order_groups(vv if order else None)
            key = "morton" if order else "ascending"
            row[f"store_{key}_ms"] = round(timed(lambda: plan.assemble_async(var, store, vals, sid, symmetric=True),
                                                 a.steps, scrub, stream), 4)
            row[f"packed_{key}_ms"] = round(timed(lambda: plan.assemble_packed_async(var, g, vals, None, sid),
                                                  a.steps, scrub, stream), 4)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
