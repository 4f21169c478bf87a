"""Where does the time between the CUDA events go for a ~20 us kernel?

Compares, for the default workload:
  single      events around one launch after an L2 flush (bench.py's method)
  graph       the same launch replayed from a captured CUDA graph
  b2b         20 back-to-back launches between one event pair (per launch)
  empty       events around an empty stream interval (timer floor)
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1103_0066_b200 as fb  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def main():
    w = sys.argv[1] if len(sys.argv) > 1 else "2d-elasticity-1m"
    prec = sys.argv[2] if len(sys.argv) > 2 else "f32"
    op, dim, ne, _ = bench.WORKLOADS[w]
    v, c, _ = bench.build_rank_mesh(op, dim, ne, 0, 1)
    var = fb.make_variant(op, dim, prec)
    dv, dc = torch.from_numpy(v).cuda(), torch.from_numpy(c).cuda()
    out = torch.empty(var.store_length(ne), device="cuda", dtype=torch.float32 if prec == "f32" else torch.float64)
    st = torch.empty(2, dtype=torch.int64, device="cuda")
    scrub = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    scrub.fill_(1)
    s = torch.cuda.Stream()
    res = {}
    with torch.cuda.stream(s):
        sid = s.cuda_stream
        fb.status_reset(st, sid)
        for _ in range(5):
            fb.integrate_mesh_async(var, dv, dc, out, st, sid)
        torch.cuda.synchronize()

        def single(n=20):
            t = []
            for _ in range(n):
                scrub.view(torch.int64).sum()
                a, b = ev(), ev()
                a.record(s)
                fb.integrate_mesh_async(var, dv, dc, out, st, sid)
                b.record(s)
                torch.cuda.synchronize()
                t.append(a.elapsed_time(b) * 1e3)
            return statistics.median(t)

        res["single_us"] = single()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fb.integrate_mesh_async(var, dv, dc, out, st, s.cuda_stream)
        t = []
        for _ in range(20):
            scrub.view(torch.int64).sum()
            a, b = ev(), ev()
            a.record(s)
            g.replay()
            b.record(s)
            torch.cuda.synchronize()
            t.append(a.elapsed_time(b) * 1e3)
        res["graph_us"] = statistics.median(t)
        scrub.view(torch.int64).sum()
        a, b = ev(), ev()
        a.record(s)
        for _ in range(20):
            fb.integrate_mesh_async(var, dv, dc, out, st, sid)
        b.record(s)
        torch.cuda.synchronize()
        res["b2b_per_launch_us"] = a.elapsed_time(b) * 1e3 / 20
        t = []
        for _ in range(20):
            scrub.view(torch.int64).sum()
            a, b = ev(), ev()
            a.record(s)
            b.record(s)
            torch.cuda.synchronize()
            t.append(a.elapsed_time(b) * 1e3)
        res["empty_us"] = statistics.median(t)
        fb.status_check(st, sid)
    res.update(workload=w, prec=prec)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
