"""Global CSR assembly timing against the HBM roofline.

    python tools/asmbench.py [--workloads 3d-laplacian-16m,2d-elasticity-1m] [--precisions f32,f64]

Per workload: the element store is produced on the device by the fused
integration kernel, then the assembly kernel is timed with CUDA events on
its stream (L2 flushed between steps by a 512 MB read outside the events).
Algorithmic bytes per launch: the incidence lists (4 + nb bytes per
incidence, nb per element) + row-block offsets (2 x 8 bytes per vertex) +
the store's real elements read once (ne * krows^2 * s) + the CSR values
written once (nnz * s).  Writes one JSON line per case and
gpurun_out/asmbench.json.
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1103_0066_b200 as fb  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--workloads", default="3d-laplacian-16m,2d-elasticity-1m,3d-elasticity-8m")
    p.add_argument("--precisions", default="f32,f64")
    p.add_argument("--steps", type=int, default=10)
    a = p.parse_args()
    peak, peak_src = bench.peaks()
    scrub = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    scrub.fill_(1)
    st = torch.empty(2, dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream()
    sid = stream.cuda_stream
    res = []
    for w in a.workloads.split(","):
        op, dim, ne, _ = bench.WORKLOADS[w]
        v, c, _ = bench.build_rank_mesh(op, dim, ne, 0, 1)
        nv = v.size // dim
        os.environ["FB_PLAN_HOST"] = "1"  # the multithreaded host builder
        t0 = time.perf_counter()
        fb.AssemblyPlan(op, dim, c, nv)
        t_plan_host = time.perf_counter() - t0
        del os.environ["FB_PLAN_HOST"]
        fb.AssemblyPlan(op, dim, c, nv)  # warm-up of the upload + GPU build path
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fb.AssemblyPlan(op, dim, c, nv)  # host cells: uploaded, planned on the GPU
        t_plan_hostcells = time.perf_counter() - t0
        dv, dc = torch.from_numpy(v).cuda(), torch.from_numpy(c).cuda()
        fb.AssemblyPlan(op, dim, dc, nv)  # warm-up (CUDA context, pools)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan = fb.AssemblyPlan(op, dim, dc, nv)  # built on the GPU
        t_plan = time.perf_counter() - t0
        nb = dim + 1
        kr = fb.engine.make_form_spec(op, dim).krows
        for prec in a.precisions.split(","):
            var = fb.make_variant(op, dim, prec, "strict")
            s = 4 if prec == "f32" else 8
            store = torch.empty(var.store_length(ne), device="cuda",
                                dtype=torch.float32 if prec == "f32" else torch.float64)
            fb.status_reset(st, sid)
            fb.integrate_mesh_async(var, dv, dc, store, st, sid)
            fb.status_check(st, sid)
            vals = torch.empty(plan.nnz, device="cuda", dtype=store.dtype)
            # elasticity also with the block-diagonal promise (SURVEY 8a row A9:
            # only block (0,0) of each element matrix is read)
            for diag in ((False, True) if op == "elasticity" else (False,)):
                for _ in range(3):
                    plan.assemble_async(var, store, vals, sid, symmetric=True, block_diagonal=diag)
                ms = []
                for _ in range(a.steps):
                    scrub.view(torch.int64).sum()
                    torch.cuda._sleep(bench.GAP_CYCLES)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    plan.assemble_async(var, store, vals, sid, symmetric=True, block_diagonal=diag)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    ms.append(e0.elapsed_time(e1))
                t = statistics.median(ms)
                read_scalars = nb * nb if diag else kr * kr
                by = ne * nb * (4 + nb) + 2 * 8 * (nv + 1) + ne * read_scalars * s + plan.nnz * s
                r = {"workload": w, "kernel": "fb_assemble_kernel" + (" (block diagonal)" if diag else ""),
                     "op": op, "dim": dim, "prec": prec,
                     "elements": ne, "rows": plan.rows, "nnz": plan.nnz, "ms": round(t, 4),
                     "algorithmic_bytes": by, "GBs": round(by / (t * 1e-3) * 1e-9),
                     "frac": round(by / (t * 1e-3) * 1e-9 / peak, 3), "peak_GBs": peak, "peak_source": peak_src,
                     "Gnnz_s": round(plan.nnz / (t * 1e-3) * 1e-9, 2),
                     "Gelem_s": round(ne / (t * 1e-3) * 1e-9, 2), "plan_build_gpu_s": round(t_plan, 4),
                     "plan_build_host_s": round(t_plan_host, 3),
                     "plan_build_from_host_cells_s": round(t_plan_hostcells, 4)}
                print(json.dumps(r), flush=True)
                res.append(r)
            # assembly straight from packed G (no element store), and the two
            # mesh -> CSR pipelines: integrate + assemble vs pack + assemble_packed
            g = torch.empty(var.store_length(ne) // (kr * kr) * dim * dim, device="cuda", dtype=store.dtype)
            fb.pack_geometry_async(dv, dc, dim, g, st, var.config.element_batch_size, prec, sid)
            pv = torch.empty_like(vals)

            def timed(fn):
                for _ in range(3):
                    fn()
                ms = []
                for _ in range(a.steps):
                    scrub.view(torch.int64).sum()
                    torch.cuda._sleep(bench.GAP_CYCLES)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    fn()
                    e1.record(stream)
                    torch.cuda.synchronize()
                    ms.append(e0.elapsed_time(e1))
                return statistics.median(ms)

            tp = timed(lambda: plan.assemble_packed_async(var, g, pv, None, sid))
            assert torch.equal(pv, vals), "packed assembly differs from the store assembly"
            t_store_path = timed(lambda: (fb.integrate_mesh_async(var, dv, dc, store, st, sid),
                                          plan.assemble_async(var, store, vals, sid, symmetric=True,
                                                              block_diagonal=op == "elasticity")))
            t_packed_path = timed(lambda: (fb.pack_geometry_async(dv, dc, dim, g, st, var.config.element_batch_size,
                                                                  prec, sid),
                                           plan.assemble_packed_async(var, g, pv, None, sid)))
            byp = ne * nb * (4 + nb) + 2 * 8 * (nv + 1) + ne * dim * dim * s + plan.nnz * s
            r = {"workload": w, "kernel": "fb_assemble_g_kernel", "op": op, "dim": dim, "prec": prec,
                 "ms": round(tp, 4), "algorithmic_bytes": byp, "GBs": round(byp / (tp * 1e-3) * 1e-9),
                 "frac": round(byp / (tp * 1e-3) * 1e-9 / peak, 3),
                 "Gelem_s": round(ne / (tp * 1e-3) * 1e-9, 2),
                 "mesh_to_csr_ms": {"integrate+assemble": round(t_store_path, 4),
                                    "pack+assemble_packed": round(t_packed_path, 4)}}
            print(json.dumps(r), flush=True)
            res.append(r)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "asmbench.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
