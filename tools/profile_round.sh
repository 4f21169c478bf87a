#!/bin/bash
# One profiling pass on the GPU box (1 GPU):  bash tools/profile_round.sh <tag>
# bench lines for every BASELINE config (each with the reference CPU
# baseline on the same mesh), the reference arm, HBM probe, the launch list
# of the default bench command, and one `ncu --set full` capture per
# (workload, precision) of the fused kernel plus the assembly / pack kernels.
# Summaries are made locally with tools/ncu_summary.py and copied to profiles/.
tag=${1:-r02}
o=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $o/${tag}_smi.txt
# fused-kernel captures first: their DRAM traffic (profiles/ncu_traffic.json,
# keyed by the kernel-source hash) feeds the bench lines' roofline block
args=""
for w in 3d-laplacian-16m 2d-elasticity-1m 3d-elasticity-8m; do
  for p in f32 f64; do
    timeout 300 ncu --set full --clock-control none --import-source on -k regex:fb_integrate_sparse -s 1 -c 1 \
        -o $o/${tag}_ncu_${w}_${p} python tools/run_kernel.py --workload $w --precision $p --reps 2 > /dev/null 2>&1
    args="$args $w:$p:strict $o/${tag}_ncu_${w}_${p}.ncu-rep"
  done
done
python tools/ncu_traffic.py $args > /dev/null && cp profiles/ncu_traffic.json $o/${tag}_ncu_traffic.json
timeout 900 python bench.py > $o/${tag}_bench_default.json 2> $o/${tag}_bench_default.err
for w in 2d-elasticity-1m 3d-elasticity-8m 2d-laplacian-64k; do
  timeout 900 python bench.py --workload $w > $o/${tag}_bench_$w.json 2> $o/${tag}_bench_$w.err
done
timeout 900 python bench.py --impl reference > $o/${tag}_bench_impl_reference.json 2> $o/${tag}_bench_ref.err
timeout 300 python tools/hbm_probe.py $o/${tag}_hbm_probe.json > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/${tag}_launches_bench_default.csv \
    python bench.py --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fb_assemble_kernel -s 1 -c 1 \
    -o $o/${tag}_ncu_assemble_3d-laplacian-16m_f32 python tools/asmbench.py --workloads 3d-laplacian-16m --precisions f32 --steps 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fb_assemble_kernel -s 1 -c 1 \
    -o $o/${tag}_ncu_assemble_3d-elasticity-8m_f64 python tools/asmbench.py --workloads 3d-elasticity-8m --precisions f64 --steps 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fb_assemble_g_kernel -s 1 -c 1 \
    -o $o/${tag}_ncu_assemble_packed_3d-elasticity-8m_f32 python tools/asmbench.py --workloads 3d-elasticity-8m --precisions f32 --steps 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:fb_integrate_sparse<float, .int.3, .int.3," -s 1 -c 1 \
    -o $o/${tag}_ncu_pack_geometry_3d_f32 python tools/pathbench.py --precisions f32 --steps 1 > /dev/null 2>&1
timeout 500 python tools/asmbench.py > $o/${tag}_asmbench.txt 2>&1
timeout 500 python tools/pathbench.py > $o/${tag}_pathbench.txt 2>&1
timeout 300 python tools/kbench.py --modes strict,fast --steps 20 > $o/${tag}_kbench.txt 2>&1
