#!/bin/bash
# ncu capture of the codec kernels (one GPU).  Usage: scripts/prof_kernels.sh <tag> [n]
set -e
TAG=${1:-r1}
N=${2:-67108864}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python scripts/kernel_timing.py --n $N > /dev/null
for K in sums encode_tiles decode_ring; do
  ncu --set full --clock-control none --import-source on -k regex:${K}_kernel -s 5 -c 1 \
      -o gpurun_out/prof_${TAG}_$K -f python scripts/kernel_timing.py --n $N > /dev/null
done
