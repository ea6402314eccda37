set -x
timeout 400 python bench.py > gpurun_out/bench_r2g.json 2> gpurun_out/bench_r2g.err
timeout 300 python bench.py --workload sweep --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2g_sweep.json 2> gpurun_out/r2g_sweep.err
timeout 300 python bench.py --workload grad_mix --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2g_gradmix.json 2> gpurun_out/r2g_gradmix.err
timeout 900 bash scripts/prof_bench.sh r2g > gpurun_out/prof_r2g.log 2>&1
echo done
