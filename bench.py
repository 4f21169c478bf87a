"""Benchmark: P1 element integration on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME]
                    [--precision f32|f64] [--mode strict|fast] [--impl ours|reference]

A step is one pass of the fused integration kernel over the rank's element
range (weak scaling: every rank owns one full copy of the workload's element
count, a contiguous slice of one global structured mesh; no collective on the
data path).  Default workload = the largest single-GPU config of BASELINE.json,
configs[2]: P1 Laplacian, 3D tetrahedra, 16,777,216 elements, FP32 strict
(bitwise the reference), with the FP64 leg in the same line and configs[1]
(2D elasticity, 1M elements, FP32 + FP64) as an extra leg.

value  = whole-job paper-count GFLOP/s (reference flop_count), device time from
         CUDA events around each kernel on the launching stream, max over ranks;
         inputs resident in HBM, L2 flushed (512 MB read) between steps.
e2e    = the same metric through the public C ABI (fb_integrate_mesh) with
         pinned HOST buffers: H2D of coordinates + connectivity, kernel, D2H of
         the full element-matrix store, every step.
--impl reference: the unmodified reference CPU engine (oracle/_ref, compiled
         from /root/reference by oracle/Makefile) on this host's cores, rank 0
         only, on the same mesh (built by the reference's own
         structured_simplicial_mesh + jitter_mesh) and the same config dict.
         This arm never loads the engine library.
--gpus N without torchrun re-launches itself under torch.distributed.run with
         N ranks; N larger than the visible GPU count is an error.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# ~100 us device-side spin before each timed launch (outside the events)
GAP_CYCLES = 200_000
SEED, JITTER, JITTER_MAX_ELEMENTS = 42, 0.15, 1 << 24
L2_BYTES = 126 << 20

WORKLOADS = {
    # name: (op, dim, elements per GPU, BASELINE.json config string)
    "3d-laplacian-16m": ("laplacian", 3, 1 << 24, "P1 Laplacian, 3D tetrahedra, 16M elements on 1 B200"),
    "2d-elasticity-1m": ("elasticity", 2, 1 << 20,
                         "P1 linear elasticity, 2D triangles, 1M elements, FP32 and FP64"),
    "2d-laplacian-64k": ("laplacian", 2, 1 << 16,
                         "P1 Laplacian, 2D triangles, 65,536 elements (CPU reference oracle run)"),
    "3d-elasticity-8m": ("elasticity", 3, 1 << 23,
                         "P1 linear elasticity, 3D tetrahedra, 64M elements sharded over 8xB200 (per-GPU shard)"),
}
DEFAULT_WORKLOAD = "3d-laplacian-16m"
EXTRA_LEG = "2d-elasticity-1m"
METRIC = "element-integration GFLOP/s and elements/s vs HBM roofline at 1/2/4/8 B200"
FALLBACK_HBM_GBS = 6650.0
# sources that determine the fused kernel's DRAM traffic (profiles/ncu_traffic.json is keyed to them)
KERNEL_SOURCES = ["fb_kernels.cuh", "fb_launch.cuh", "fb_internal.h", "fb_kernels_f32_2d.cu",
                  "fb_kernels_f32_3d.cu", "fb_kernels_f64_2d.cu", "fb_kernels_f64_3d.cu"]


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    p.add_argument("--precision", default="f32", choices=["f32", "f64"])
    p.add_argument("--mode", default="strict", choices=["strict", "fast"])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--e2e-steps", type=int, default=10)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-assembly", action="store_true", help="skip the global CSR assembly leg")
    p.add_argument("--no-extra-leg", action="store_true", help=f"skip the {EXTRA_LEG} leg")
    return p.parse_args(argv)


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


def mesh_resolution(dim, num_elements):
    """Smallest n whose structured mesh (reference geometry.cpp:164-234:
    2n^2 triangles / 6n^3 tetrahedra) has >= num_elements cells."""
    n = 1
    while (2 * n * n if dim == 2 else 6 * n ** 3) < num_elements:
        n += 1
    return n


def jitter_for(total):
    # the reference's jitter_mesh validates every cell serially: applied where
    # affordable, values change but bytes and flops do not
    return JITTER if total <= JITTER_MAX_ELEMENTS else 0.0


def step_traffic(op, dim, elements, prec):
    """Connectivity + store bytes of one step (the vertices add ~4-8 B/element)."""
    s = 4 if prec == "f32" else 8
    return elements * (dim + 1) * 4 + elements * krows(op, dim) ** 2 * s


def workload_config(name, prec, mode, world):
    """The config dict both arms print, byte for byte."""
    op, dim, ne_per, cfg_name = WORKLOADS[name]
    total = ne_per * world
    step_bytes = step_traffic(op, dim, total, prec)
    return {"workload": name, "baseline_config": cfg_name, "op": op, "dim": dim,
            "elements": total, "elements_per_gpu": ne_per,
            "mesh": f"first {total} cells of structured_simplicial_mesh(dim={dim}, n={mesh_resolution(dim, total)})",
            "jitter": jitter_for(total), "seed": SEED, "precision": prec, "mode": mode,
            "element_batch_size": 128, "parallelism": f"element shards x{world}, no collectives",
            "l2": (f"flushed between steps (512 MB read outside the events); per-step traffic "
                   f"{step_bytes / 1e9:.2f} GB {'>' if step_bytes > L2_BYTES else '<'} 126 MB L2")}


def build_rank_mesh_engine(op, dim, ne_per, rank, world):
    """Our arm: the reference mesh synthesised by the engine library
    (bit-identical to the reference's, tests/test_abi.py)."""
    from paper_1103_0066_b200 import mesh_prefix

    total = ne_per * world
    v, c, n = mesh_prefix(dim, total, jitter_for(total), SEED)
    assert n == mesh_resolution(dim, total)
    nb = dim + 1
    return v, np.ascontiguousarray(c[rank * ne_per * nb:(rank + 1) * ne_per * nb]), n


def build_rank_mesh_reference(dim, ne_per, rank, world):
    """Reference arm: the reference's own structured_simplicial_mesh +
    jitter_mesh (oracle/_ref), never the engine library."""
    from oracle.oracle import Reference

    total = ne_per * world
    n = mesh_resolution(dim, total)
    v, c = Reference().make_mesh(dim, n, jitter_for(total), SEED)
    nb = dim + 1
    return v, np.ascontiguousarray(c[rank * ne_per * nb:(rank + 1) * ne_per * nb]), n


# kept for tools/ (kbench, pathbench, asmbench, sweep): the engine-built mesh
def build_rank_mesh(op, dim, ne_per, rank, world, jitter=None, seed=SEED):
    return build_rank_mesh_engine(op, dim, ne_per, rank, world)


def algorithmic_bytes(op, dim, prec, cells, nv_ref):
    """int32 connectivity + each referenced FP64 vertex once + the store."""
    ne = cells.size // (dim + 1)
    s = 4 if prec == "f32" else 8
    return ne * (dim + 1) * 4 + nv_ref * dim * 8 + ne * krows(op, dim) ** 2 * s


def kernel_source_sha():
    h = hashlib.sha256()
    for f in KERNEL_SOURCES:
        with open(os.path.join(ROOT, "paper_1103_0066_b200", "csrc", f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def committed_traffic(workload, prec, mode):
    """DRAM bytes per launch from the committed `ncu --set full` capture
    (profiles/ncu_traffic.json), only if it was taken on the current kernel
    sources; otherwise None (stale)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None, "no capture committed"
    with open(path) as f:
        d = json.load(f).get(f"{workload}:{prec}:{mode}")
    if not isinstance(d, dict):
        return None, "no capture for this key"
    if d.get("kernel_sha") != kernel_source_sha():
        return None, f"capture is stale (kernel sources changed since {d.get('kernel_sha')})"
    return float(d["traffic"]), d.get("report", "ncu --set full")


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


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_baseline(op, dim, prec, v, cells, target_s=20.0):
    """The reference's own CPU path (oracle/_ref) on this host's cores: the
    mesh-in / matrices-out composition pack_geometry + integrate_batches
    (reference bench.cpp:150-164, include_packing=true) with the paper's best
    variant (bs128 ce2 interleaved), workers = every host thread, over the
    FULL workload (reps bounded to ~target_s); workers = 1 as well when one
    rep is short (at 16.7M elements the serial run
    would take minutes and is never the better one).  Integrate-only timing
    (include_packing=false) is reported beside it."""
    from oracle.oracle import Reference, Restatement, reference_available

    ne = cells.size // (dim + 1)
    flops = flops_per_element(op, dim) * ne
    cores = host_cores()
    p = 0 if prec == "f32" else 1
    if reference_available():
        ref = Reference()
        kw = dict(bs=128, ce=2, interleave=True, precision=p)
        t1, _ = ref.time_integrate(op, v, cells, dim, workers=cores, reps=1, include_packing=True, **kw)
        reps = int(max(1, min(20, target_s / 2 / max(t1, 1e-6))))
        tmin, tmean = ref.time_integrate(op, v, cells, dim, workers=cores, reps=reps, include_packing=True, **kw)
        best, tried = (cores, tmin, tmean, reps), [cores]
        if t1 * cores < target_s / 4 and cores > 1:
            s1, m1 = ref.time_integrate(op, v, cells, dim, workers=1, reps=reps, include_packing=True, **kw)
            tried.append(1)
            if s1 < tmin:
                best = (1, s1, m1, reps)
        workers, tmin, tmean, reps = best
        ti, _ = ref.time_integrate(op, v, cells, dim, workers=workers, reps=max(1, reps // 2),
                                   include_packing=False, **kw)
        return {"value": flops / tmin * 1e-9, "unit": "GFLOP/s", "cores": workers, "kind": "reference",
                "elements_per_s": ne / tmin, "seconds_min": tmin, "seconds_mean": tmean,
                "integrate_only_gflops": flops / ti * 1e-9, "host_threads": cores, "cpu_model": cpu_model(),
                "sample": f"full workload ({ne} elements) x {reps} reps, pack_geometry+integrate_batches "
                          f"(reference bench.cpp:150-164), bs128 ce2 interleaved, workers={workers} "
                          f"(tried {tried}), min over reps"}
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
    """The reference's CPU implementation (oracle/_ref) on this host, same
    workload / mesh / config dict as our arm; rank 0 only (other ranks exit)."""
    if rank != 0:
        return
    from oracle.oracle import Reference, Restatement, reference_available

    op, dim, ne_per, _ = WORKLOADS[args.workload]
    cores = host_cores()
    prec = 0 if args.precision == "f32" else 1
    kind = "reference" if reference_available() else "port"
    t_mesh = time.perf_counter()
    if kind == "reference":
        v, c, _ = build_rank_mesh_reference(dim, ne_per, 0, world)
        builder = "reference structured_simplicial_mesh + jitter_mesh (oracle/_ref)"
    else:  # no reference build here: the C restatement on the (unjittered) numpy mesh
        from oracle.oracle import structured_mesh_numpy

        v, c = structured_mesh_numpy(dim, mesh_resolution(dim, ne_per * world))
        c = np.ascontiguousarray(c[: ne_per * (dim + 1)])
        builder = "oracle.structured_mesh_numpy (unjittered: jitter changes values, not work)"
    t_mesh = time.perf_counter() - t_mesh
    ne = c.size // (dim + 1)
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
    flops = flops_per_element(op, dim) * ne
    val = flops / (ms * 1e-3) * 1e-9
    shard = "" if world == 1 else f" (rank 0's shard of the {ne_per * world}-element job; CPU throughput is per host)"
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "elements_per_s": ne / (ms * 1e-3),
        "config": workload_config(args.workload, args.precision, args.mode, world),
        "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": cores if kind == "reference" else 1,
                         "kind": kind,
                         "cpu_model": cpu_model(),
                         "sample": f"{ne} elements per step{shard}: pack_geometry + integrate_batches "
                                   f"(reference bench.cpp:150-164, include_packing=true) bs128 ce2 "
                                   f"interleaved, workers={cores}, output store allocated+zeroed per call "
                                   f"(engine.cpp:215-217); mean of {args.steps} steps"},
        "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "mesh_build_s": t_mesh,
        "mesh_builder": builder,
    }
    print(json.dumps(line), flush=True)


def spawn_ranks(args):
    """--gpus N outside torchrun: re-launch this script with N ranks."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    rank, world, local = dist_env()
    if world == 1 and args.gpus > 1:
        if args.impl != "reference" and os.environ.get("FB_BENCH_SHARED_GPU") != "1":
            import torch

            if torch.cuda.device_count() < args.gpus:
                sys.exit(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs; {torch.cuda.device_count()} visible")
        sys.exit(spawn_ranks(args))
    if world > 1 and args.gpus != world:
        sys.exit(f"bench.py: --gpus {args.gpus} but torchrun started {world} ranks")
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch

    import paper_1103_0066_b200 as fb

    ndev = torch.cuda.device_count()
    shared = os.environ.get("FB_BENCH_SHARED_GPU") == "1"  # test mode: ranks share one GPU (gloo)
    if world > ndev and not shared:
        sys.exit(f"bench.py: --gpus {world} needs {world} GPUs; {ndev} visible")
    local = local % max(ndev, 1)
    torch.cuda.set_device(local)
    dist = None
    backend = None
    if world > 1:
        import torch.distributed as dist

        # one process per GPU over NCCL; gloo only when ranks share a GPU (test mode)
        backend = "nccl" if ndev >= world else "gloo"
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")

    op, dim, ne_per, _ = WORKLOADS[args.workload]
    prec = args.precision
    v, cells, n = build_rank_mesh_engine(op, dim, ne_per, rank, world)
    nv_ref = int(np.unique(cells).size)
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

    def kernel_steps(variant, vtx, cel, output, k, warm, flush=True):
        """k timed launches, each between its own CUDA events (L2 flushed before
        each) -> (mean ms, min ms, launches)."""
        fb.status_reset(status, sid)
        for _ in range(warm):
            fb.integrate_mesh_async(variant, vtx, cel, output, status, sid)
        torch.cuda.synchronize()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        barrier()
        torch.cuda.synchronize()
        n0 = fb.launch_counter()
        clocks.mark()
        for i in range(k):
            if flush:
                scrub.view(torch.int64).sum()  # flush L2 with clean lines (outside the events)
            # keep the device queue ahead of the host: the start event is then
            # stamped when the launch is already enqueued (outside the events)
            torch.cuda._sleep(GAP_CYCLES)
            starts[i].record(stream)
            fb.integrate_mesh_async(variant, vtx, cel, output, status, sid)
            ends[i].record(stream)
        torch.cuda.synchronize()
        clocks.unmark()
        barrier()
        launches = fb.launch_counter() - n0
        fb.status_check(status, sid)
        ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
        return statistics.mean(ms), min(ms), launches

    def pcie_floor(h2d_pairs, dout, hout, reps=3):
        """The copy engines' floor for one e2e step: the step's H2D copies (pinned
        -> device) and its D2H store copy on two streams at once, plus each
        direction alone -- raw torch copies, no kernel (best of `reps`)."""
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

        def run(up, down):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if up:
                with torch.cuda.stream(s1):
                    for h, d in h2d_pairs:
                        d.copy_(h, non_blocking=True)
            if down:
                with torch.cuda.stream(s2):
                    hout.copy_(dout, non_blocking=True)
            torch.cuda.synchronize()
            return time.perf_counter() - t0

        both = min(run(True, True) for _ in range(reps))
        up = min(run(True, False) for _ in range(reps))
        down = min(run(False, True) for _ in range(reps))
        nb_up = sum(h.numel() * h.element_size() for h, _ in h2d_pairs)
        nb_down = hout.numel() * hout.element_size()
        return {"ms": both * 1e3, "h2d_GBs": nb_up / up * 1e-9, "d2h_GBs": nb_down / down * 1e-9,
                "what": "the step's H2D and D2H as raw concurrent copies (no kernel); frac = this / e2e ms_per_step"}

    def back_to_back(variant, vtx, cel, output, k):
        """k launches captured in one CUDA graph and replayed inside ONE event
        pair, no flush between (device-side steady state: a Python launch loop
        would measure the host's launch rate for the small kernels)."""
        fb.status_reset(status, sid)
        fb.integrate_mesh_async(variant, vtx, cel, output, status, sid)  # set-up outside the capture
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        try:
            with torch.cuda.graph(graph, stream=cap):
                for _ in range(k):
                    fb.integrate_mesh_async(variant, vtx, cel, output, status, cap.cuda_stream)
            graph.replay()  # warm
            torch.cuda.synchronize()
        except RuntimeError:  # no graph capture here: a launch loop (host-rate bound for tiny kernels)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n0 = fb.launch_counter()
            torch.cuda._sleep(GAP_CYCLES)
            e0.record(stream)
            for _ in range(k):
                fb.integrate_mesh_async(variant, vtx, cel, output, status, sid)
            e1.record(stream)
            torch.cuda.synchronize()
            fb.status_check(status, sid)
            return e0.elapsed_time(e1) / k, fb.launch_counter() - n0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n0 = fb.launch_counter()
        clocks.mark()
        torch.cuda._sleep(GAP_CYCLES)
        e0.record(stream)
        graph.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        clocks.unmark()
        fb.status_check(status, sid)
        # the library's counter saw the k captured launches once; each replay
        # launches them again on the device
        return e0.elapsed_time(e1) / k, k + (fb.launch_counter() - n0)

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    peak, peak_src = peaks()
    flops = flops_per_element(op, dim) * ne_per * world
    with ClockSampler(local) as clocks:
        ms_mean, ms_min, launches = kernel_steps(var, dv, dc, out, args.steps, args.warmup)
        ms_mean = max_over_ranks(ms_mean)
        # steps whose traffic is within ~2x of L2: also the steady state (back to
        # back launches, no flush), as in a solver loop re-integrating one mesh
        steady = None
        if step_traffic(op, dim, ne_per * world, prec) < 2 * L2_BYTES:
            b2b, lb = back_to_back(var, dv, dc, out, args.steps)
            steady = max_over_ranks(b2b)
            launches += lb

        # e2e through the public C ABI with pinned host buffers
        hv = torch.from_numpy(v).pin_memory()
        hc = torch.from_numpy(cells).pin_memory()
        hout = torch.empty(store_len, dtype=tdt).pin_memory()
        hv_np, hc_np, hout_np = hv.numpy(), hc.numpy(), hout.numpy()
        for _ in range(2):
            fb.integrate_mesh(var, hv_np, hc_np, out=hout_np, devices=[local])
        barrier()
        n0 = fb.launch_counter()
        clocks.mark()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            fb.integrate_mesh(var, hv_np, hc_np, out=hout_np, devices=[local])
        e2e_ms = (time.perf_counter() - t0) * 1e3 / args.e2e_steps
        clocks.unmark()
        e2e_launches = fb.launch_counter() - n0
        barrier()
        e2e_ms = max_over_ranks(e2e_ms)
        pcie = pcie_floor([(hv, dv), (hc, dc)], out, hout)
        del hout, hout_np

        # the other arithmetic mode of the same precision (fast: FP64 edges, then
        # FMA geometry in the engine precision; within the stated tolerances,
        # tests/test_gpu_parity.py -- not bitwise)
        omode = "fast" if args.mode == "strict" else "strict"
        var_m = fb.make_variant(op, dim, prec, omode, element_batch_size=128)
        ms_m, _, lm = kernel_steps(var_m, dv, dc, out, args.steps, args.warmup)
        ms_m = max_over_ranks(ms_m)
        launches += lm

        # the other precision of the same config, same mesh
        other = "f64" if prec == "f32" else "f32"
        var2 = fb.make_variant(op, dim, other, args.mode, element_batch_size=128)
        out2 = torch.empty(store_len, dtype=torch.float64 if other == "f64" else torch.float32, device=dev)
        ms2, _, l2 = kernel_steps(var2, dv, dc, out2, args.steps, args.warmup)
        ms2 = max_over_ranks(ms2)
        launches += l2
        del out2

        # extra leg: BASELINE configs[1] (2D elasticity 1M, FP32 + FP64), flushed
        # and back to back (its f32 store is ~1.2x L2: steady state differs)
        extra = None
        if not args.no_extra_leg and args.workload != EXTRA_LEG:
            eop, edim, ene, _ = WORKLOADS[EXTRA_LEG]
            ev, ec, _ = build_rank_mesh_engine(eop, edim, ene, rank, world)
            env_ref = int(np.unique(ec).size)
            edv, edc = torch.from_numpy(ev).to(dev), torch.from_numpy(ec).to(dev)
            extra = {"config": workload_config(EXTRA_LEG, "f32", args.mode, world)}
            for p in ("f32", "f64"):
                evar = fb.make_variant(eop, edim, p, args.mode, element_batch_size=128)
                eout = torch.empty(evar.store_length(ene), device=dev,
                                   dtype=torch.float32 if p == "f32" else torch.float64)
                m, _, l_ = kernel_steps(evar, edv, edc, eout, args.steps, args.warmup)
                b2b, lb = back_to_back(evar, edv, edc, eout, args.steps)
                m, b2b = max_over_ranks(m), max_over_ranks(b2b)
                launches += l_ + lb
                eb = algorithmic_bytes(eop, edim, p, ec, env_ref)
                ef = flops_per_element(eop, edim) * ene * world
                extra[p] = {"value": ef / (m * 1e-3) * 1e-9, "unit": "GFLOP/s", "ms_per_step": m,
                            "elements_per_s": ene * world / (m * 1e-3),
                            "roofline_frac": eb / (m * 1e-3) * 1e-9 / peak,
                            "back_to_back": {"ms_per_launch": b2b, "value": ef / (b2b * 1e-3) * 1e-9,
                                             "roofline_frac": eb / (b2b * 1e-3) * 1e-9 / peak,
                                             "note": f"{args.steps} launches in one CUDA graph replayed inside one event pair, no L2 flush"}}
                del eout
            del edv, edc

        # global CSR assembly of the timed store (device-resident)
        asm = None
        if not args.no_assembly:
            plan = fb.AssemblyPlan(op, dim, dc, v.size // dim)  # plan built on the GPU
            vals = torch.empty(plan.nnz, dtype=tdt, device=dev)
            sym = var.path in (0, 3)
            # elasticity from a P1-sparse variant: block-diagonal element matrices
            # with equal diagonal blocks, only block (0,0) read
            diag = op == "elasticity" and var.path != 2

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

            fb.integrate_mesh_async(var, dv, dc, out, status, sid)
            asm = {"nnz": plan.nnz}
            asm["ms"], asm["launches"] = dev_timed(
                lambda: plan.assemble_async(var, out, vals, sid, symmetric=sym, block_diagonal=diag))
            asm["block_diagonal"] = diag
            g = torch.empty(store_len // (krows(op, dim) ** 2) * dim * dim, dtype=tdt, device=dev)
            gst = torch.empty(2, dtype=torch.int64, device=dev)
            fb.pack_geometry_async(dv, dc, dim, g, gst, 128, prec, sid)
            pvals = torch.empty_like(vals)
            asm["packed_ms"], asm["packed_launches"] = dev_timed(
                lambda: plan.assemble_packed_async(var, g, pvals, None, sid))
            if args.mode == "strict" and not torch.equal(pvals, vals):  # strict: mesh path == G path
                raise RuntimeError("packed-geometry assembly differs from the store assembly")
            asm["pipe_store_ms"], l3 = dev_timed(lambda: (fb.integrate_mesh_async(var, dv, dc, out, gst, sid),
                                                       plan.assemble_async(var, out, vals, sid, symmetric=sym,
                                                                           block_diagonal=diag)))
            asm["pipe_packed_ms"], l4 = dev_timed(lambda: (fb.pack_geometry_async(dv, dc, dim, g, gst, 128, prec, sid),
                                                        plan.assemble_packed_async(var, g, pvals, None, sid)))
            asm["pipe_launches"] = l3 + l4
            del g, pvals, vals, plan

    torch.cuda.synchronize()

    value = flops / (ms_mean * 1e-3) * 1e-9
    bytes_launch = algorithmic_bytes(op, dim, prec, cells, nv_ref)
    achieved = bytes_launch / (ms_mean * 1e-3) * 1e-9
    bytes2 = algorithmic_bytes(op, dim, other, cells, nv_ref)
    traffic, traffic_src = committed_traffic(args.workload, prec, args.mode)
    h2d = v.nbytes + cells.nbytes
    d2h = store_len * (4 if prec == "f32" else 8) + 16
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
            "peak_source": peak_src, "algorithmic_bytes_per_launch": bytes_launch,
            "algorithmic_bytes_per_element": bytes_launch / ne_per,
            "kernel": "fb_integrate_sparse (fused geometry + G:K + staged stores)"}
    if traffic:
        roof["traffic_over_algorithmic"] = traffic / bytes_launch
        roof["dram_frac"] = traffic / (ms_mean * 1e-3) * 1e-9 / peak  # DRAM-true fraction

    line = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_mean, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": prec, "data": "synthetic",
        "elements_per_s": ne_per * world / (ms_mean * 1e-3),
        "config": workload_config(args.workload, prec, args.mode, world),
        "roofline": roof,
        "e2e": {"value": flops / (e2e_ms * 1e-3) * 1e-9, "unit": "GFLOP/s", "ms_per_step": e2e_ms,
                "elements_per_s": ne_per * world / (e2e_ms * 1e-3),
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "gpu_launches": e2e_launches,
                "pcie_floor": dict(pcie, frac=pcie["ms"] / e2e_ms),
                "api": "fb_integrate_mesh (C ABI), pinned host buffers, chunked H2D/kernel/D2H pipeline"},
        "gpu_launches": launches,
        other: {"value": flops / (ms2 * 1e-3) * 1e-9, "unit": "GFLOP/s", "ms_per_step": ms2,
                "elements_per_s": ne_per * world / (ms2 * 1e-3),
                "roofline_frac": bytes2 / (ms2 * 1e-3) * 1e-9 / peak},
        "ms_min": ms_min,
        f"{prec}_{omode}": {"value": flops / (ms_m * 1e-3) * 1e-9, "unit": "GFLOP/s", "ms_per_step": ms_m,
                            "roofline_frac": bytes_launch / (ms_m * 1e-3) * 1e-9 / peak,
                            "parity": ("normwise <= 5e-6 (f32) / 1e-13 (f64) vs the FP64 direct oracle"
                                       if omode == "fast" else "bitwise the reference")},
        "steady_state": None if steady is None else {
            "ms_per_launch": steady, "value": flops / (steady * 1e-3) * 1e-9,
            "roofline_frac": bytes_launch / (steady * 1e-3) * 1e-9 / peak,
            "note": f"{args.steps} launches in one CUDA graph replayed inside one event pair, no L2 flush "
                    f"(step traffic < 2x L2)"},
        "run": {"dist_backend": backend, "mesh_builder": "engine (fb_structured_mesh + fb_jitter_mesh, "
                                                         "bit-identical to the reference's)"},
    }
    if extra is not None:
        line["legs"] = {EXTRA_LEG: extra}
    if asm is not None:
        s_ = 4 if prec == "f32" else 8
        nb_ = dim + 1
        kr = krows(op, dim)
        nv_all = v.size // dim
        read_scalars = nb_ * nb_ if asm["block_diagonal"] else kr * kr
        a_bytes = ne_per * nb_ * (4 + nb_) + 2 * 8 * (nv_all + 1) + ne_per * read_scalars * s_ + asm["nnz"] * s_
        a_ach = a_bytes / (asm["ms"] * 1e-3) * 1e-9
        line["assembly"] = {
            "kernel": "fb_assemble_kernel (deterministic CSR gather, SURVEY 8f F3)"
                      + (", block-diagonal reads" if asm["block_diagonal"] else ""), "ms_per_step": asm["ms"],
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
        line["gpu_launches"] += asm["launches"] + asm["packed_launches"] + asm["pipe_launches"]
    line["clocks"] = clocks.summary()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(op, dim, prec, v, cells)
        if args.workload == "3d-elasticity-8m":
            line["cpu_baseline"]["sample"] += ("; this is configs[3]'s per-GPU shard (1/8 of the 64M-element job): "
                                               "the reference's 64M time is 8x this shard's at the same GFLOP/s")
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
