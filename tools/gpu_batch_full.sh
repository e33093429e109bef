#!/bin/bash
# full GPU suite (all ranks the box has), probe, launch times of the solve, c4 bench
T=${1:-full}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
timeout 300 python tools/perf_probe.py --solve 1 > gpurun_out/${T}_probe.log 2>&1
timeout 600 bash tools/ncu_times.sh "." ${T}_all.csv
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench_c4.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_c4.log
