#!/bin/bash
# ncu: launch list + full capture of the warp-run encoder (one GPU)
TAG=${1:-w1}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_encw_$TAG.csv \
    python scripts/exp/encode_only_time.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:encode_warps_kernel -s 4 -c 1 \
    -o gpurun_out/prof_encw_$TAG -f python scripts/exp/encode_only_time.py > /dev/null 2>&1
echo done
