#!/bin/bash
# ncu --set full of one decode_ring_kernel launch at the layer size (one GPU)
set -e
TAG=${1:-dec}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:decode_ring -s 3 -c 1 \
    -o gpurun_out/prof_$TAG -f python scripts/exp/decode_time.py > /dev/null
