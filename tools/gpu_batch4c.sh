#!/bin/bash
# 4-GPU: per-phase z-slab timings (dist_probe) at 1/2/4 ranks with both exchange paths, c4 bench at 4.
T=${1:-b4c}
mkdir -p gpurun_out
for x in nccl peer; do
  for n in 1 2 4; do
    EXCHANGE=$x timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 2990$n tools/dist_probe.py >> gpurun_out/${T}_probe.log 2>&1
  done
done
for x in nccl peer; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29814 \
    bench.py --gpus 4 --steps 10 --warmup 3 --exchange $x --no-fp64-line > gpurun_out/${T}_bench_c4_n4_$x.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_c4_n4_$x.log
done
