"""Per-step device times of the bench's timed loop in three enqueue modes
(back to back, synchronised per step, back to back with a device-side gap
before each start event): shows host launch latency leaking into the first
back-to-back step.  python tools/steps_probe.py"""
import statistics, sys, json
sys.path.insert(0, ".")
import torch, bench
import paper_1103_0066_b200 as fb
op, dim, ne, _ = bench.WORKLOADS["2d-elasticity-1m"]
v, c, _ = bench.build_rank_mesh(op, dim, ne, 0, 1)
dv, dc = torch.from_numpy(v).cuda(), torch.from_numpy(c).cuda()
var = fb.make_variant(op, dim, "f32", "strict")
out = torch.empty(var.store_length(ne), device="cuda")
st = torch.empty(2, dtype=torch.int64, device="cuda")
scrub = torch.empty(512 << 20, dtype=torch.uint8, device="cuda"); scrub.fill_(1)
s = torch.cuda.current_stream(); sid = s.cuda_stream
for _ in range(5): fb.integrate_mesh_async(var, dv, dc, out, st, sid)
torch.cuda.synchronize()
for mode in ["b2b", "sync", "b2b+gap", "b2b", "b2b+gap"]:
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    for a, b in ev:
        scrub.view(torch.int64).sum()
        if mode.endswith("gap"): torch.cuda._sleep(bench.GAP_CYCLES)
        a.record(s); fb.integrate_mesh_async(var, dv, dc, out, st, sid); b.record(s)
        if mode == "sync": torch.cuda.synchronize()
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) * 1000 for a, b in ev]
    print(mode, "mean %.1f median %.1f min %.1f" % (statistics.mean(ms), statistics.median(ms), min(ms)), [round(x, 1) for x in ms])
