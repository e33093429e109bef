#!/bin/bash
# 4-GPU batch: distributed parity (peer + NCCL exchanges), c4 bench at 2 and 4 GPUs, c5 at 4.
T=${1:-b4b}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_dist_gpu.py -q -p no:cacheprovider -s -x > gpurun_out/${T}_dist_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_dist_tests.log
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2970$n \
    bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/${T}_bench_c4_n$n.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_c4_n$n.log
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29724 \
  bench.py --config c5 --gpus 4 --steps 3 --warmup 3 --no-fp64-line > gpurun_out/${T}_bench_c5_n4.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_c5_n4.log
