#!/bin/bash
# Round-2 evidence run on one B200: the non-headline bench workloads, the
# N>1 code paths with ranks sharing the GPU, and the loud --gpus N failure.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python bench.py --workload sweep --steps 10 --warmup 3 > gpurun_out/r2_sweep.json 2> gpurun_out/r2_sweep.err
timeout 300 python bench.py --workload grad_mix --steps 10 --warmup 3 > gpurun_out/r2_gradmix.json 2> gpurun_out/r2_gradmix.err
python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/r2_gpus2_on_1gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_gpus2_on_1gpu.txt
for w in layer_ag moe_a2a imbalance; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29533 \
    bench.py --gpus 2 --share-gpu --backend gloo --workload $w --tokens 1024 --steps 5 --warmup 3 --no-cpu-baseline \
    > gpurun_out/r2_share2_$w.json 2> gpurun_out/r2_share2_$w.err
done
echo done
