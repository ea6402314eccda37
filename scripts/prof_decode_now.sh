#!/bin/bash
# ncu --set full of the decoder at the layer size (scripts/exp/decode_time.py)
TAG=${1:-d1}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:decode_ring -s 3 -c 1 \
    -o gpurun_out/prof_dec_$TAG -f python scripts/exp/decode_time.py > /dev/null 2>&1
echo done
