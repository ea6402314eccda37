#!/bin/bash
# ncu evidence for the bench step (one GPU): launch list + full capture of the top kernels.
set -e
TAG=${1:-r1}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --clock-settle 0 --no-graph > gpurun_out/bench_under_ncu_$TAG.json
# encode_tiles launches alternate <1> (the fused encoder) / <0> (the no-op
# conditional re-encode), so an even skip count lands on the fused encoder
for K in decode_ring encode_tiles encode_runfix guess_kernel; do
  F=$K
  ncu --set full --clock-control none --import-source on -k regex:"$K" -s 4 -c 1 \
      -o gpurun_out/prof_bench_${TAG}_$F -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --clock-settle 0 --no-graph > /dev/null
done
