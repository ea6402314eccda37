#!/bin/bash
# Final round-2 evidence on one B200: headline bench line, C5 sweep, C4 mixes,
# ncu launch list + full captures of the bench kernels (scripts/prof_bench.sh).
mkdir -p gpurun_out
set -x
timeout 400 python bench.py > gpurun_out/bench_r2h.json 2> gpurun_out/bench_r2h.err
timeout 300 python bench.py --workload sweep --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2h_sweep.json 2> gpurun_out/r2h_sweep.err
timeout 300 python bench.py --workload grad_mix --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2h_gradmix.json 2> gpurun_out/r2h_gradmix.err
timeout 900 bash scripts/prof_bench.sh r2h > gpurun_out/prof_r2h.log 2>&1
echo done
