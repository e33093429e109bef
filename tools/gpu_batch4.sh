#!/bin/bash
# 4-GPU batch: distributed parity tests, 1-GPU kernel probe, bench at 1/2/4 GPUs (c4) and c5 at 1/4.
T=${1:-b4}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_dist_gpu.py tests/test_dist_gloo.py -q -p no:cacheprovider -s > gpurun_out/${T}_dist_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_dist_tests.log
timeout 300 python tools/perf_probe.py --solve 1 > gpurun_out/${T}_probe.log 2>&1
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n \
    bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/${T}_bench_c4_n$n.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_c4_n$n.log
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29614 \
  bench.py --config c5 --gpus 4 --steps 3 --warmup 3 --no-fp64-line > gpurun_out/${T}_bench_c5_n4.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_c5_n4.log
timeout 1500 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-fp64-line > gpurun_out/${T}_bench_c5_n1.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_c5_n1.log
