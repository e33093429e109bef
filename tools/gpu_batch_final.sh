#!/bin/bash
# Final check on a 4-GPU box: the whole GPU suite (the 2- and 4-rank tests included), the c4
# bench at 1/2/4 GPUs with the default (peer) exchanges, c5 at 4 GPUs, smoke().
T=${1:-final}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1; echo rc=$? >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench_c4_n1.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_c4_n1.log
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2980$n \
    bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/${T}_bench_c4_n$n.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_c4_n$n.log
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${T}_bench_ref.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_ref.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29814 \
  bench.py --config c5 --gpus 4 --steps 3 --warmup 3 --no-fp64-line > gpurun_out/${T}_bench_c5_n4.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_c5_n4.log
