#!/bin/bash
# 2-GPU A/B of the z-slab exchange paths (c4 bench) + the 2-rank parity tests.
T=${1:-b2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dist_gpu.py -q -p no:cacheprovider -k "2-4" > gpurun_out/${T}_dist_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_dist_tests.log
for x in nccl peer; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2980${#x} \
    bench.py --gpus 2 --steps 10 --warmup 3 --exchange $x --no-fp64-line > gpurun_out/${T}_bench_c4_n2_$x.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_c4_n2_$x.log
done
