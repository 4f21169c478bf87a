"""Small runs of every kernel path, for compute-sanitizer (memcheck /
racecheck / synccheck):

    compute-sanitizer --tool memcheck --error-exitcode 1 python tools/sanitize_run.py

Covers the fused integration (every op x dim x precision x store path,
ragged tile counts, unaligned output), GPU pack_geometry, the G-input path,
the GPU assembly plan build and both assembly kernels (store and packed G,
incl. hub vertices beyond the shared-memory slots, and the block-diagonal
store reads).  Run with
PYTORCH_NO_CUDA_MEMORY_CACHING=1 so every buffer is its own allocation.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1103_0066_b200 as fb  # noqa: E402


def main():
    st = torch.empty(2, dtype=torch.int64, device="cuda")
    sid = torch.cuda.current_stream().cuda_stream
    for dim, n in ((2, 5), (3, 2)):
        v, c = fb.structured_mesh(dim, n, 0.1, 7)
        ne = c.size // (dim + 1)
        dv, dc = torch.from_numpy(v).cuda(), torch.from_numpy(c).cuda()
        w = torch.from_numpy(np.ascontiguousarray(1.0 + v.reshape(-1, dim)[c.reshape(-1, dim + 1), 0].ravel())).cuda()
        for prec in ("f32", "f64"):
            dt = torch.float32 if prec == "f32" else torch.float64
            for op in ("laplacian", "elasticity", "weighted-laplacian"):
                coeffs = w if op == "weighted-laplacian" else None
                for mode in ("strict", "fast"):
                    for store in ("auto", "staged", "tma", "direct"):
                        var = fb.make_variant(op, dim, prec, mode, element_batch_size=8, store=store)
                        out = torch.empty(var.store_length(ne) + 1, dtype=dt, device="cuda")
                        for o in (out[:-1], out[1:]):  # aligned and unaligned stores
                            fb.status_reset(st, sid)
                            fb.integrate_mesh_async(var, dv, dc, o, st, sid, coefficients=coeffs)
                            fb.status_check(st, sid)
                var = fb.make_variant(op, dim, prec, "strict", element_batch_size=8)
                g = torch.empty(var.store_length(ne) // var.spec.krows ** 2 * dim * dim, dtype=dt, device="cuda")
                fb.pack_geometry_async(dv, dc, dim, g, st, 8, prec, sid)
                out = torch.empty(var.store_length(ne), dtype=dt, device="cuda")
                fb.integrate_packed_async(var, g, ne, out, sid, coefficients=coeffs)
                plan = fb.AssemblyPlan(op, dim, dc, v.size // dim)
                for sym in (False, True):
                    for diag in ((False, True) if op == "elasticity" else (False,)):
                        vals = torch.empty(plan.nnz, dtype=dt, device="cuda")
                        plan.assemble_async(var, out, vals, sid, symmetric=sym, block_diagonal=diag)
                # assembly from packed G: G of exactly ne*dim^2 scalars (the
                # vector loads' tail guard), aligned and misaligned
                gx = torch.empty(ne * dim * dim + 1, dtype=dt, device="cuda")
                for gg in (gx[:-1], gx[1:]):
                    gg.copy_(g[: ne * dim * dim])
                    plan.assemble_packed_async(var, gg, vals, coeffs, sid)
                torch.cuda.synchronize()
    # hub vertices beyond the shared-memory slots (global accumulation paths)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_gpu_assembly import fan_mesh

    for dim in (2, 3):
        v, c = fan_mesh(dim, 40)
        ne = c.size // (dim + 1)
        dv, dc = torch.from_numpy(v).cuda(), torch.from_numpy(c).cuda()
        for prec in ("f32", "f64"):
            dt = torch.float32 if prec == "f32" else torch.float64
            for op in ("laplacian", "elasticity"):
                var = fb.make_variant(op, dim, prec, "strict", element_batch_size=8)
                g = torch.empty(var.store_length(ne) // var.spec.krows ** 2 * dim * dim, dtype=dt, device="cuda")
                fb.pack_geometry_async(dv, dc, dim, g, st, 8, prec, sid)
                out = torch.empty(var.store_length(ne), dtype=dt, device="cuda")
                fb.integrate_packed_async(var, g, ne, out, sid)
                plan = fb.AssemblyPlan(op, dim, dc, v.size // dim)
                vals = torch.empty(plan.nnz, dtype=dt, device="cuda")
                plan.assemble_async(var, out, vals, sid, symmetric=True)
                if op == "elasticity":
                    plan.assemble_async(var, out, vals, sid, symmetric=True, block_diagonal=True)
                plan.assemble_packed_async(var, g, vals, None, sid)
                torch.cuda.synchronize()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
