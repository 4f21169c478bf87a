"""Benchmark: P1 element integration on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME]
                    [--precision f32|f64] [--mode strict|fast] [--impl ours|reference]

A step is one pass of the fused integration kernel over the rank's element
range (weak scaling: every rank owns one full copy of the workload's element
count, a contiguous slice of one global structured mesh; no collective on the
data path).  Default workload = BASELINE.json configs[1]: P1 linear
elasticity, 2D triangles, 1,048,576 elements, FP32 (FP64 reported alongside).

value  = whole-job paper-count GFLOP/s (reference flop_count), device time from
         CUDA events around each kernel on the launching stream, max over ranks;
         inputs resident in HBM, L2 flushed (512 MB read) between steps.
e2e    = the same metric through the public C ABI (fb_integrate_mesh) with
         pinned HOST buffers: H2D of coordinates + connectivity, kernel, D2H of
         the full element-matrix store, every step.
assembly = global CSR assembly of the timed store on the
         device: kernel time from CUDA events, its own HBM roofline.
--impl reference: the unmodified reference CPU engine (oracle/_ref, built from
         /root/reference) on this host's cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# ~100 us device-side spin before each timed launch (outside the events)
GAP_CYCLES = 200_000

WORKLOADS = {
    # name: (op, dim, elements per GPU, BASELINE.json config string)
    "2d-elasticity-1m": ("elasticity", 2, 1 << 20,
                         "P1 linear elasticity, 2D triangles, 1M elements, FP32 and FP64"),
    "2d-laplacian-64k": ("laplacian", 2, 1 << 16,
                         "P1 Laplacian, 2D triangles, 65,536 elements (CPU reference oracle run)"),
    "3d-laplacian-16m": ("laplacian", 3, 1 << 24, "P1 Laplacian, 3D tetrahedra, 16M elements on 1 B200"),
    "3d-elasticity-8m": ("elasticity", 3, 1 << 23,
                         "P1 linear elasticity, 3D tetrahedra, 64M elements sharded over 8xB200 (per-GPU shard)"),
}
METRIC = "element-integration GFLOP/s and elements/s vs HBM roofline at 1/2/4/8 B200"
FALLBACK_HBM_GBS = 6650.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--workload", default="2d-elasticity-1m", choices=sorted(WORKLOADS))
    p.add_argument("--precision", default="f32", choices=["f32", "f64"])
    p.add_argument("--mode", default="strict", choices=["strict", "fast"])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--e2e-steps", type=int, default=10)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-assembly", action="store_true", help="skip the global CSR assembly leg")
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def krows(op, dim):
    return (dim + 1) * dim if op == "elasticity" else dim + 1


def flops_per_element(op, dim):
    kr, dd = krows(op, dim), dim * dim
    return kr * kr * 2 * dd if op != "weighted-laplacian" else kr * kr * (dim + 1) * (2 * dd + 2)


def build_rank_mesh(op, dim, ne_per, rank, world, jitter=0.15, seed=42):
    """Slice [rank*ne, (rank+1)*ne) of the first world*ne cells of the
    reference structured mesh (jittered where the reference would afford it)."""
    from paper_1103_0066_b200 import mesh_prefix

    total = ne_per * world
    v, c, n = mesh_prefix(dim, total, jitter if total <= (1 << 24) else 0.0, seed)
    nb = dim + 1
    cells = np.ascontiguousarray(c[rank * ne_per * nb:(rank + 1) * ne_per * nb])
    return v, cells, n


def algorithmic_bytes(op, dim, prec, cells, nv_ref):
    ne = cells.size // (dim + 1)
    s = 4 if prec == "f32" else 8
    return ne * (dim + 1) * 4 + nv_ref * dim * 8 + ne * krows(op, dim) ** 2 * s


class ClockSampler:
    """SM clock and throttle reasons sampled through NVML (nvidia-ml-py) every
    ~2 ms; mark()/unmark() bracket the timed regions so the summary reflects
    the clocks the measured kernels actually ran at."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, device_index: int):
        self.dev = device_index
        self.samples = []  # (in_timed_region, sm_mhz, reasons_mask)
        self.timed = False
        self.stop = threading.Event()
        self.max_mhz = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.dev)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def poll():
                while not self.stop.is_set():
                    try:
                        mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((self.timed, mhz, rs))
                    except Exception:
                        pass
                    time.sleep(0.002)

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
        except Exception:
            self.t = None
        return self

    def mark(self):
        self.timed = True

    def unmark(self):
        self.timed = False

    def __exit__(self, *a):
        self.stop.set()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        timed = [s for s in self.samples if s[0]] or self.samples
        if not timed:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        mask = 0
        for s in timed:
            mask |= s[2]
        return {"sm_mhz": statistics.median(s[1] for s in timed), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(k for k, bit in self.REASONS.items() if mask & bit),
                "samples": len(timed), "source": "nvml 2 ms polling inside the timed regions"}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(op, dim, prec, v, cells, target_s=10.0):
    """The reference's own CPU path (oracle/_ref) on this host's cores: the
    mesh-in / matrices-out composition pack_geometry + integrate_batches with
    the paper's best variant (bs128 ce2 interleaved); workers = all hardware
    threads and 1, the better reported, plus the
    reference's integrate-only timing (include_packing=false) for context."""
    from oracle.oracle import Reference, Restatement, reference_available

    ne = cells.size // (dim + 1)
    flops = flops_per_element(op, dim) * ne
    cores = os.cpu_count() or 1
    p = 0 if prec == "f32" else 1
    if reference_available():
        ref = Reference()
        best = None
        for workers in sorted({cores, 1}, reverse=True):
            t1, _ = ref.time_integrate(op, v, cells, dim, bs=128, ce=2, interleave=True, precision=p,
                                       workers=workers, reps=1, include_packing=True)
            reps = int(max(1, min(50, target_s / 2 / max(t1, 1e-6))))
            tmin, tmean = ref.time_integrate(op, v, cells, dim, bs=128, ce=2, interleave=True, precision=p,
                                             workers=workers, reps=reps, include_packing=True)
            if best is None or tmin < best[1]:
                best = (workers, tmin, tmean, reps)
        workers, tmin, tmean, reps = best
        ti, _ = ref.time_integrate(op, v, cells, dim, bs=128, ce=2, interleave=True, precision=p,
                                   workers=workers, reps=max(1, reps // 2), include_packing=False)
        return {"value": flops / tmin * 1e-9, "unit": "GFLOP/s", "cores": workers, "kind": "reference",
                "elements_per_s": ne / tmin, "seconds_min": tmin, "seconds_mean": tmean,
                "integrate_only_gflops": flops / ti * 1e-9, "host_threads": cores, "cpu_model": cpu_model(),
                "sample": f"full workload ({ne} elements) x {reps} reps, pack_geometry+integrate_batches, "
                          f"bs128 ce2 interleaved, workers={workers} (best of {cores} and 1), min over reps"}
    ora = Restatement()
    sample = min(ne, 1 << 18)
    c = np.ascontiguousarray(cells[: sample * (dim + 1)])
    t0 = time.perf_counter()
    ora.integrate_mesh(op, v, c, dim, bs=128, precision=prec)
    t = time.perf_counter() - t0
    return {"value": flops_per_element(op, dim) * sample / t * 1e-9, "unit": "GFLOP/s", "cores": 1,
            "kind": "port", "elements_per_s": sample / t, "cpu_model": cpu_model(),
            "sample": f"first {sample} elements, C restatement, 1 thread"}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    op, dim, ne_per, cfg_name = WORKLOADS[args.workload]
    from oracle.oracle import Reference, Restatement, reference_available

    total = ne_per * world
    sample = min(total, 1 << 22)
    v, c, _ = build_rank_mesh(op, dim, sample, 0, 1)
    cores = os.cpu_count() or 1
    prec = 0 if args.precision == "f32" else 1
    kind = "reference" if reference_available() else "port"
    times = []
    for i in range(args.warmup + args.steps):
        if kind == "reference":
            t, _ = Reference().time_integrate(op, v, c, dim, bs=128, ce=2, interleave=True, precision=prec,
                                              workers=cores, reps=1, include_packing=True)
        else:
            t0 = time.perf_counter()
            Restatement().integrate_mesh(op, v, c, dim, bs=128, precision=prec)
            t = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(t)
    ms = statistics.mean(times) * 1e3
    flops = flops_per_element(op, dim) * sample
    val = flops / (ms * 1e-3) * 1e-9
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "elements_per_s": sample / (ms * 1e-3),
        "config": {"workload": args.workload, "baseline_config": cfg_name, "elements": total,
                   "sampled_elements": sample, "precision": args.precision, "parallelism": "cpu threads"},
        "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": cores if kind == "reference" else 1,
                         "kind": kind,
                         "sample": f"{sample} of {total} elements per step; pack_geometry+integrate_batches "
                                   f"bs128 ce2 interleaved"},
        "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch

    import paper_1103_0066_b200 as fb

    ndev = torch.cuda.device_count()
    local = local % max(ndev, 1)  # >1 rank per GPU only when testing the N>1 path on a 1-GPU box
    torch.cuda.set_device(local)
    dist = None
    backend = None
    if world > 1:
        import torch.distributed as dist

        # one process per GPU over NCCL; gloo only if ranks outnumber GPUs (test mode)
        backend = "nccl" if ndev >= world else "gloo"
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")

    op, dim, ne_per, cfg_name = WORKLOADS[args.workload]
    prec = args.precision
    v, cells, n = build_rank_mesh(op, dim, ne_per, rank, world)
    nv_ref = int(np.unique(cells).size)
    kr = krows(op, dim)
    var = fb.make_variant(op, dim, prec, args.mode, element_batch_size=128)
    store_len = var.store_length(ne_per)

    dev = torch.device("cuda", local)
    dv = torch.from_numpy(v).to(dev)
    dc = torch.from_numpy(cells).to(dev)
    tdt = torch.float32 if prec == "f32" else torch.float64
    out = torch.empty(store_len, dtype=tdt, device=dev)
    status = torch.empty(2, dtype=torch.int64, device=dev)
    scrub = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    scrub.fill_(1)
    stream = torch.cuda.current_stream()
    sid = stream.cuda_stream

    def barrier():
        if dist is not None:
            dist.barrier()

    def kernel_steps(variant, output, k, warm):
        fb.status_reset(status, sid)
        for _ in range(warm):
            fb.integrate_mesh_async(variant, dv, dc, output, status, sid)
        torch.cuda.synchronize()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        barrier()
        torch.cuda.synchronize()
        n0 = fb.launch_counter()
        clocks.mark()
        for i in range(k):
            scrub.view(torch.int64).sum()  # flush L2 with clean lines (outside the events)
            # keep the device queue ahead of the host: the start event is then
            # stamped when the launch is already enqueued, so no host launch
            # latency lands inside the device-timed window (outside the events)
            torch.cuda._sleep(GAP_CYCLES)
            starts[i].record(stream)
            fb.integrate_mesh_async(variant, dv, dc, output, status, sid)
            ends[i].record(stream)
        torch.cuda.synchronize()
        clocks.unmark()
        barrier()
        launches = fb.launch_counter() - n0
        fb.status_check(status, sid)
        ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
        return statistics.mean(ms), min(ms), launches

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    with ClockSampler(local) as clocks:
        ms_mean, ms_min, launches = kernel_steps(var, out, args.steps, args.warmup)
        ms_mean = max_over_ranks(ms_mean)

        # e2e through the public C ABI with pinned host buffers
        hv = torch.from_numpy(v).pin_memory()
        hc = torch.from_numpy(cells).pin_memory()
        hout = torch.empty(store_len, dtype=tdt).pin_memory()
        hv_np, hc_np, hout_np = hv.numpy(), hc.numpy(), hout.numpy()
        for _ in range(2):
            fb.integrate_mesh(var, hv_np, hc_np, out=hout_np, devices=[local])
        barrier()
        clocks.mark()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            fb.integrate_mesh(var, hv_np, hc_np, out=hout_np, devices=[local])
        e2e_ms = (time.perf_counter() - t0) * 1e3 / args.e2e_steps
        clocks.unmark()
        barrier()
        e2e_ms = max_over_ranks(e2e_ms)

        # the FP64 leg of the same config (BASELINE configs[1] asks for both)
        other = "f64" if prec == "f32" else "f32"
        var2 = fb.make_variant(op, dim, other, args.mode, element_batch_size=128)
        out2 = torch.empty(store_len, dtype=torch.float64 if other == "f64" else torch.float32, device=dev)
        ms2, _, l2 = kernel_steps(var2, out2, args.steps, args.warmup)
        ms2 = max_over_ranks(ms2)
        launches += l2

        # global CSR assembly of the timed store (device-resident)
        asm = None
        if not args.no_assembly:
            plan = fb.AssemblyPlan(op, dim, dc, v.size // dim)  # plan built on the GPU
            vals = torch.empty(plan.nnz, dtype=tdt, device=dev)
            for _ in range(max(args.warmup, 1)):
                plan.assemble_async(var, out, vals, sid, symmetric=var.path in (0, 3))
            torch.cuda.synchronize()
            barrier()
            a_ms = []
            na0 = fb.launch_counter()
            clocks.mark()
            for _ in range(args.steps):
                scrub.view(torch.int64).sum()
                torch.cuda._sleep(GAP_CYCLES)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                plan.assemble_async(var, out, vals, sid, symmetric=var.path in (0, 3))
                e1.record(stream)
                torch.cuda.synchronize()
                a_ms.append(e0.elapsed_time(e1))
            clocks.unmark()
            barrier()
            asm = {"ms": max_over_ranks(statistics.mean(a_ms)), "nnz": plan.nnz,
                   "launches": fb.launch_counter() - na0}

            # the same operator straight from packed geometry (no element store),
            # and the two mesh -> CSR pipelines end to end on the device
            def dev_timed(fn):
                for _ in range(max(args.warmup, 1)):
                    fn()
                torch.cuda.synchronize()
                barrier()
                ms = []
                n0 = fb.launch_counter()
                clocks.mark()
                for _ in range(args.steps):
                    scrub.view(torch.int64).sum()
                    torch.cuda._sleep(GAP_CYCLES)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    fn()
                    e1.record(stream)
                    torch.cuda.synchronize()
                    ms.append(e0.elapsed_time(e1))
                clocks.unmark()
                barrier()
                return max_over_ranks(statistics.mean(ms)), fb.launch_counter() - n0

            g = torch.empty(store_len // (kr * kr) * dim * dim, dtype=tdt, device=dev)
            gst = torch.empty(2, dtype=torch.int64, device=dev)
            fb.pack_geometry_async(dv, dc, dim, g, gst, 128, prec, sid)
            pvals = torch.empty_like(vals)
            asm["packed_ms"], asm["packed_launches"] = dev_timed(
                lambda: plan.assemble_packed_async(var, g, pvals, None, sid))
            if args.mode == "strict" and not torch.equal(pvals, vals):  # strict: mesh path == G path
                raise RuntimeError("packed-geometry assembly differs from the store assembly")
            asm["pipe_store_ms"], _ = dev_timed(lambda: (fb.integrate_mesh_async(var, dv, dc, out, gst, sid),
                                                      plan.assemble_async(var, out, vals, sid,
                                                                          symmetric=var.path in (0, 3))))
            asm["pipe_packed_ms"], _ = dev_timed(lambda: (fb.pack_geometry_async(dv, dc, dim, g, gst, 128, prec, sid),
                                                       plan.assemble_packed_async(var, g, pvals, None, sid)))

    # parity spot check of the timed output (full bitwise check lives in tests/)
    torch.cuda.synchronize()

    flops = flops_per_element(op, dim) * ne_per * world
    value = flops / (ms_mean * 1e-3) * 1e-9
    peak, peak_src = peaks()
    bytes_launch = algorithmic_bytes(op, dim, prec, cells, nv_ref)
    achieved = bytes_launch / (ms_mean * 1e-3) * 1e-9
    bytes2 = algorithmic_bytes(op, dim, other, cells, nv_ref)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get(f"{args.workload}:{prec}:{args.mode}")
    h2d = v.nbytes + cells.nbytes
    d2h = store_len * (4 if prec == "f32" else 8) + 16

    line = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_mean, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": prec, "data": "synthetic",
        "elements_per_s": ne_per * world / (ms_mean * 1e-3),
        "config": {"workload": args.workload, "baseline_config": cfg_name, "op": op, "dim": dim,
                   "elements_per_gpu": ne_per, "elements": ne_per * world, "mesh": f"structured n={n} prefix",
                   "jitter": 0.15 if ne_per * world <= (1 << 24) else 0.0, "precision": prec,
                   "mode": args.mode, "parallelism": f"element shards x{world}, no collectives",
                   "dist_backend": backend,
                   "l2": "flushed between steps (512 MB read, outside the events)",
                   "element_batch_size": 128},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": bytes_launch,
                     "kernel": "fb_integrate_sparse (fused geometry + G:K + staged stores)"},
        "e2e": {"value": flops / (e2e_ms * 1e-3) * 1e-9, "unit": "GFLOP/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "fb_integrate_mesh (C ABI), pinned host buffers"},
        "gpu_launches": launches,
        other: {"value": flops / (ms2 * 1e-3) * 1e-9, "ms_per_step": ms2,
                "elements_per_s": ne_per * world / (ms2 * 1e-3),
                "roofline_frac": bytes2 / (ms2 * 1e-3) * 1e-9 / peak},
        "ms_min": ms_min,
        "clocks": clocks.summary(),
    }
    if asm is not None:
        s_ = 4 if prec == "f32" else 8
        nb_ = dim + 1
        nv_all = v.size // dim
        a_bytes = ne_per * nb_ * (4 + nb_) + 2 * 8 * (nv_all + 1) + ne_per * kr * kr * s_ + asm["nnz"] * s_
        a_ach = a_bytes / (asm["ms"] * 1e-3) * 1e-9
        line["assembly"] = {
            "kernel": "fb_assemble_kernel (deterministic CSR gather, SURVEY 8f F3)", "ms_per_step": asm["ms"],
            "nnz_per_gpu": asm["nnz"], "Gnnz_per_s": asm["nnz"] * world / (asm["ms"] * 1e-3) * 1e-9,
            "roofline": {"bound": "hbm", "achieved": a_ach, "peak": peak, "unit": "GB/s", "frac": a_ach / peak,
                         "algorithmic_bytes_per_launch": a_bytes},
            "gpu_launches": asm["launches"]}
        p_bytes = ne_per * nb_ * (4 + nb_) + 2 * 8 * (nv_all + 1) + ne_per * dim * dim * s_ + asm["nnz"] * s_
        p_ach = p_bytes / (asm["packed_ms"] * 1e-3) * 1e-9
        line["assembly"]["from_packed_geometry"] = {
            "kernel": "fb_assemble_g_kernel (element rows recomputed from packed G, no element store)",
            "ms_per_step": asm["packed_ms"],
            "roofline": {"bound": "hbm", "achieved": p_ach, "peak": peak, "unit": "GB/s", "frac": p_ach / peak,
                         "algorithmic_bytes_per_launch": p_bytes},
            "gpu_launches": asm["packed_launches"]}
        line["assembly"]["mesh_to_csr_ms"] = {"integrate_mesh+assemble": asm["pipe_store_ms"],
                                              "pack_geometry+assemble_packed": asm["pipe_packed_ms"]}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(op, dim, prec, v, cells)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
