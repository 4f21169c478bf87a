"""Element-count sweep (BASELINE.json configs[4]): N = 2^12 ... 2^28 elements
for {Laplacian, elasticity} x {2D, 3D} x {f32, f64}, strict mode, on G GPUs of
this process (the engine's contiguous tile-aligned element shards,
fb.shard_bounds, one per device, no collectives).  Inputs resident, L2
flushed between steps.  ms = (G > 1) wall time from a host barrier (all
devices idle) to the last device's completion, launches issued by one host
thread per device, or (G = 1) the kernel's CUDA-event time;
ms_device_max = max over devices of the CUDA-event kernel time.  The same
points are also written in the reference's benchmark-record CSV schema plus
the SURVEY section 5 extension columns (devices, gbytes_per_s,
roofline_fraction, ref_cpu_seconds = the reference CPU path on all host
threads for N <= 2^22, host_cores) to profiles/<out>_records.csv.  Writes CSV rows to stdout and to
profiles/<out>.csv.

    python tools/sweep.py [--gpus G] [--min-log2 12] [--max-log2 28] [--step 2] [--out r01_sweep_1gpu]

Meshes are prefixes of the reference structured mesh (unjittered: jitter
changes values, not bytes or flops).  Points whose per-GPU store exceeds
--max-store-gb are skipped (3D elasticity f64 at 2^28 needs 309 GB).
"""
import argparse
import csv
import os
import shutil
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1103_0066_b200 as fb  # noqa: E402
import threading  # noqa: E402
import time  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--min-log2", type=int, default=12)
    p.add_argument("--max-log2", type=int, default=28)
    p.add_argument("--step", type=int, default=2)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--max-store-gb", type=float, default=120.0)
    p.add_argument("--ops", default="laplacian,elasticity")
    p.add_argument("--dims", default="2,3")
    p.add_argument("--precisions", default="f32,f64")
    p.add_argument("--out", default="r02_sweep_1gpu")
    p.add_argument("--ref-max-log2", type=int, default=22,
                   help="time the reference CPU path (oracle/_ref, all host threads) up to this size")
    p.add_argument("--checksum-max-log2", type=int, default=24)
    a = p.parse_args()
    peak, _ = bench.peaks()
    G = min(a.gpus, torch.cuda.device_count())
    scrubs = [torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{d}") for d in range(G)]
    for s in scrubs:
        s.fill_(1)
    fields = ["op", "dim", "precision", "elements", "gpus", "ms", "ms_device_max", "gbytes_per_s", "roofline_fraction",
              "gflops", "gelem_per_s", "status"]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    path = os.path.join(ROOT, "profiles", a.out + ".csv")
    f = open(path, "w", newline="")
    w = csv.DictWriter(f, fieldnames=fields)
    w.writeheader()
    # the same points in the reference's benchmark-record schema (src/bench.cpp
    # CSV, 15 columns) plus the extension columns of SURVEY section 5
    records = []
    EXT = ("devices", "gbytes_per_s", "roofline_fraction", "ref_cpu_seconds", "host_cores")
    host_cores = bench.host_cores()
    try:
        from oracle.oracle import Reference, reference_available
        ref = Reference() if reference_available() else None
    except Exception:
        ref = None
    sizes = [1 << k for k in range(a.min_log2, a.max_log2 + 1, a.step)]
    for dim in [int(x) for x in a.dims.split(",")]:
        v, c, _ = fb.mesh_prefix(dim, sizes[-1], 0.0, 42)
        nb = dim + 1
        for N in sizes:
            cN = c[: N * nb]
            nv_ref = int(np.unique(cN).size) if N <= (1 << 24) else int(cN.max()) + 1
            for op in a.ops.split(","):
                for prec in a.precisions.split(","):
                    kr = bench.krows(op, dim)
                    s = 4 if prec == "f32" else 8
                    row = {"op": op, "dim": dim, "precision": prec, "elements": N, "gpus": G}
                    rec = {"operator": op, "dim": dim, "num_elements": N, "batch_size": 128, "concurrent": 1,
                           "interleave": False, "unroll": False, "precision": prec, "workers": G,
                           "reps": a.steps, "seconds_min": 0.0, "seconds_mean": 0.0, "gflops": 0.0,
                           "checksum": 0.0, "devices": G, "host_cores": host_cores}
                    if N * kr * kr * s / G > a.max_store_gb * 1e9:
                        row["status"] = "skipped: store exceeds per-GPU budget"
                        rec["status"] = row["status"]
                        records.append(rec)
                        w.writerow(row)
                        f.flush()
                        print(row, flush=True)
                        continue
                    var = fb.make_variant(op, dim, prec)
                    b = fb.shard_bounds(N, G)
                    shards = []
                    for d in range(G):
                        with torch.cuda.device(d):
                            cs = torch.from_numpy(np.ascontiguousarray(cN[b[d] * nb:b[d + 1] * nb])).cuda(d)
                            vs = torch.from_numpy(v).cuda(d)
                            out = torch.empty(var.store_length(b[d + 1] - b[d]), device=f"cuda:{d}",
                                              dtype=torch.float32 if prec == "f32" else torch.float64)
                            st = torch.empty(2, dtype=torch.int64, device=f"cuda:{d}")
                            shards.append((vs, cs, out, st))
                    times, dev_times = [], []
                    for it in range(2 + a.steps):
                        evs = [None] * G
                        for d in range(G):  # flush every L2 first (outside the timed window)
                            with torch.cuda.device(d):
                                scrubs[d].view(torch.int64).sum()
                                if it == 0:
                                    fb.status_reset(shards[d][3], torch.cuda.current_stream().cuda_stream)
                        for d in range(G):
                            torch.cuda.synchronize(d)
                        go = threading.Barrier(G + 1)

                        def run(d):
                            torch.cuda.set_device(d)
                            sid = torch.cuda.current_stream().cuda_stream
                            vs, cs, out, st = shards[d]
                            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                            go.wait()
                            # keep the device queue ahead of the host so the start
                            # event is not stamped before the (Python) launch
                            if G == 1:
                                torch.cuda._sleep(bench.GAP_CYCLES)
                            e0.record()
                            if cs.numel():
                                fb.integrate_mesh_async(var, vs, cs, out, st, sid)
                            e1.record()
                            e1.synchronize()
                            evs[d] = (e0, e1)

                        pool = [threading.Thread(target=run, args=(d,)) for d in range(G)]
                        for t in pool:
                            t.start()
                        go.wait()
                        t0 = time.perf_counter()
                        for t in pool:
                            t.join()
                        wall = (time.perf_counter() - t0) * 1e3
                        if it >= 2:
                            dev = max(e0.elapsed_time(e1) for e0, e1 in evs)
                            # one device: its kernel time (a host wall clock around a
                            # ~3 us kernel is thread wake-up and launch latency)
                            times.append(wall if G > 1 else dev)
                            dev_times.append(dev)
                    for d in range(G):
                        with torch.cuda.device(d):
                            fb.status_check(shards[d][3], torch.cuda.current_stream().cuda_stream)
                    # checksum: real entries in element order, summed sequentially in double
                    csum = float("nan")
                    if N <= (1 << a.checksum_max_log2):
                        kr2 = kr * kr
                        tot = 0.0
                        for d in range(G):
                            o = shards[d][2][: (b[d + 1] - b[d]) * kr2].double().cpu().numpy()
                            for q in range(0, o.size, 1 << 24):
                                cs = np.cumsum(np.concatenate(([tot], o[q:q + (1 << 24)])))
                                tot = float(cs[-1])
                        csum = tot
                    ref_s = None
                    if ref is not None and N <= (1 << a.ref_max_log2):
                        ref_s, _ = ref.time_integrate(op, v, cN, dim, bs=128, ce=2, interleave=True,
                                                      precision=0 if prec == "f32" else 1, workers=host_cores,
                                                      reps=1, include_packing=True)
                    del shards
                    ms = statistics.median(times)
                    by = N * nb * 4 + nv_ref * dim * 8 + N * kr * kr * s
                    gbs = by / (ms * 1e-3) * 1e-9
                    row.update(ms=round(ms, 5), ms_device_max=round(statistics.median(dev_times), 5),
                               gbytes_per_s=round(gbs, 1),
                               roofline_fraction=round(gbs / (peak * G), 4),
                               gflops=round(bench.flops_per_element(op, dim) * N / (ms * 1e-3) * 1e-9, 1),
                               gelem_per_s=round(N / (ms * 1e-3) * 1e-9, 3), status="ok")
                    w.writerow(row)
                    f.flush()
                    print(row, flush=True)
                    rec.update(seconds_min=min(times) * 1e-3, seconds_mean=statistics.mean(times) * 1e-3,
                               gflops=bench.flops_per_element(op, dim) * N / (min(times) * 1e-3) * 1e-9,
                               checksum=csum, gbytes_per_s=gbs, roofline_fraction=gbs / (peak * G),
                               ref_cpu_seconds=ref_s, status="ok")
                    records.append(rec)
    f.close()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    rpath = os.path.join(ROOT, "profiles", a.out + "_records.csv")
    fb.write_bench_csv(rpath, records, extra=EXT)
    shutil.copy(rpath, os.path.join(ROOT, "gpurun_out", a.out + "_records.csv"))
    # a copy the GPU-box runner brings back
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    shutil.copy(path, os.path.join(ROOT, "gpurun_out", a.out + ".csv"))
    print("wrote", path)


if __name__ == "__main__":
    main()
