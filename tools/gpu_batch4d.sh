#!/bin/bash
# 4-GPU batch: distributed parity tests, c4 at 2/4 GPUs (NCCL and peer exchange), c5 at 4 and 1,
# c2/c3 at 1 GPU.
T=${1:-b4d}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_dist_gpu.py tests/test_dist_gloo.py -q -p no:cacheprovider > gpurun_out/${T}_dist_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_dist_tests.log
for n in 2 4; do
  for x in nccl peer; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2970$n \
      bench.py --gpus $n --steps 10 --warmup 3 --exchange $x --no-fp64-line > gpurun_out/${T}_bench_c4_n${n}_$x.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_c4_n${n}_$x.log
  done
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29714 \
  bench.py --config c5 --gpus 4 --steps 3 --warmup 3 --no-fp64-line > gpurun_out/${T}_bench_c5_n4.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_c5_n4.log
for c in c2 c3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${T}_bench_$c.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_$c.log
done
timeout 1500 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-fp64-line > gpurun_out/${T}_bench_c5_n1.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_c5_n1.log
