#!/bin/bash
# face-pass A/B (row-list grid, blocks per launch), launch times, parity subset, c4 bench
T=${1:-r}
mkdir -p gpurun_out
for v in "" fb16; do
  if [ -z "$v" ]; then lib=libsemlab_b200.so; else lib=libsemlab_b200_$v.so; fi
  SEMLAB_LIB=$lib timeout 300 python tools/perf_probe.py --solve 1 > gpurun_out/${T}_probe_${v:-default}.log 2>&1
done
timeout 300 bash tools/ncu_times.sh "k_pass|k_face|k_axe|k_rasw" ${T}_times.csv
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "space or pmg or scale or steady or dist" \
  > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench_c4.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_c4.log
