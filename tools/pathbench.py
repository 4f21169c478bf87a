"""Kernel timing of the SURVEY 8f "next" paths against the HBM roofline:
F1 weighted Laplacian (fused, per-element P1 coefficients), F2 the G-input
path (integrate_batches on packed G) and the GPU pack_geometry kernel.

    python tools/pathbench.py [--precisions f32,f64] [--steps 10]

CUDA events on the launching stream, median of --steps, L2 flushed between
steps (512 MB read outside the events).  Algorithmic bytes per launch:
  weighted fused : ne*nb*4 (cells) + nv_ref*dim*8 (vertices) + ne*nb*8 (coefficients) + ne*krows^2*s
  packed         : nslots*dim^2*s (G) + nslots*krows^2*s (store)
  pack_geometry  : ne*nb*4 + nv_ref*dim*8 + nslots*dim^2*s (G)
Writes one JSON line per case and gpurun_out/pathbench.json.
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

CASES = [  # (path, op, dim, elements)
    ("weighted-fused", "weighted-laplacian", 2, 1 << 20),
    ("weighted-fused", "weighted-laplacian", 3, 1 << 24),
    ("packed", "elasticity", 2, 1 << 20),
    ("packed", "laplacian", 3, 1 << 24),
    ("pack_geometry", None, 2, 1 << 20),
    ("pack_geometry", None, 3, 1 << 24),
    # the 2D launch-size effect: the same kernels at 16M elements
    ("weighted-fused", "weighted-laplacian", 2, 1 << 24),
    ("pack_geometry", None, 2, 1 << 24),
]


def main():
    p = argparse.ArgumentParser()
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
    meshes = {}
    for path, op, dim, ne in CASES:
        if (dim, ne) not in meshes:
            v, c, _ = bench.build_rank_mesh("laplacian", dim, ne, 0, 1)
            meshes[(dim, ne)] = (v, c, int(np.unique(c).size))
        v, c, nv_ref = meshes[(dim, ne)]
        dv, dc = torch.from_numpy(v).cuda(), torch.from_numpy(c).cuda()
        nb, dd = dim + 1, dim * dim
        nslots = -(-ne // 128) * 128
        for prec in a.precisions.split(","):
            s = 4 if prec == "f32" else 8
            tdt = torch.float32 if prec == "f32" else torch.float64
            if path == "weighted-fused":
                var = fb.make_variant(op, dim, prec, "strict")
                w = torch.from_numpy(1.0 + v.reshape(-1, dim)[c.reshape(-1, nb), 0].ravel()).cuda()
                out = torch.empty(var.store_length(ne), dtype=tdt, device="cuda")
                run = lambda: fb.integrate_mesh_async(var, dv, dc, out, st, sid, coefficients=w)  # noqa: E731
                kr = var.spec.krows
                by = ne * nb * 4 + nv_ref * dim * 8 + ne * nb * 8 + ne * kr * kr * s
                flops = bench.flops_per_element(op, dim) * ne
            elif path == "packed":
                var = fb.make_variant(op, dim, prec, "strict")
                g = torch.empty(nslots * dd, dtype=tdt, device="cuda")
                fb.status_reset(st, sid)
                fb.pack_geometry_async(dv, dc, dim, g, st, 128, prec, sid)
                out = torch.empty(var.store_length(ne), dtype=tdt, device="cuda")
                run = lambda: fb.integrate_packed_async(var, g, ne, out, sid)  # noqa: E731
                kr = var.spec.krows
                by = nslots * dd * s + nslots * kr * kr * s
                flops = bench.flops_per_element(op, dim) * ne
            else:
                g = torch.empty(nslots * dd, dtype=tdt, device="cuda")
                run = lambda: fb.pack_geometry_async(dv, dc, dim, g, st, 128, prec, sid)  # noqa: E731
                by = ne * nb * 4 + nv_ref * dim * 8 + nslots * dd * s
                flops = 0
            fb.status_reset(st, sid)
            for _ in range(3):
                run()
            ms = []
            for _ in range(a.steps):
                scrub.view(torch.int64).sum()
                torch.cuda._sleep(bench.GAP_CYCLES)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                run()
                e1.record(stream)
                torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
            fb.status_check(st, sid)
            t = statistics.median(ms)
            gbs = by / (t * 1e-3) * 1e-9
            r = {"path": path, "op": op, "dim": dim, "prec": prec, "elements": ne, "ms": round(t, 4),
                 "algorithmic_bytes": by, "GBs": round(gbs), "frac": round(gbs / peak, 3), "peak_GBs": peak,
                 "peak_source": peak_src, "Gelem_s": round(ne / (t * 1e-3) * 1e-9, 2),
                 "GFLOPs": round(flops / (t * 1e-3) * 1e-9, 1)}
            print(json.dumps(r), flush=True)
            res.append(r)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "pathbench.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
