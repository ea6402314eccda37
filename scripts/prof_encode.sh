#!/bin/bash
# ncu --set full of one fused-encoder launch (encode_tiles_kernel<1>) at the layer size
set -e
TAG=${1:-enc}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:encode_tiles -s 6 -c 1 \
    -o gpurun_out/prof_$TAG -f python scripts/exp/decode_time.py > /dev/null
