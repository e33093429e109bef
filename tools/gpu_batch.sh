#!/bin/bash
# One gpurun batch: GPU tests, bench lines for every BASELINE config, the eta sweep, the ncu launch
# list of the c4 bench. usage: tools/gpu_batch.sh TAG   (outputs gpurun_out/TAG_*)
T=${1:-batch}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench_c4.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_c4.log
for c in c1 c2 c3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${T}_bench_$c.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_$c.log
done
timeout 900 python tools/eta_sweep.py --elems 32 --out gpurun_out/${T}_eta_E32.csv > gpurun_out/${T}_eta_E32.md 2>&1
timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-fp64-line > gpurun_out/${T}_bench_c5.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_c5.log
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-fp64-line > gpurun_out/${T}_ncu_bench.log 2>&1
python tools/launch_share.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launch_share.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${T}_smi.txt
