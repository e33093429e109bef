#!/bin/bash
# A/B of variant libraries (VARIANTS="name ..." -> libsemlab_b200_<name>.so) against the default:
# probe each, launch times of each, parity subset and the c4 bench on the default.
T=${1:-r}
mkdir -p gpurun_out
for v in "" $VARIANTS; do
  if [ -z "$v" ]; then lib=libsemlab_b200.so; else lib=libsemlab_b200_$v.so; fi
  SEMLAB_LIB=$lib timeout 300 python tools/perf_probe.py --solve 1 > gpurun_out/${T}_probe_${v:-default}.log 2>&1
  SEMLAB_LIB=$lib timeout 300 bash tools/ncu_times.sh "${KERNELS:-k_pass|k_face|k_axe|k_rasw}" ${T}_times_${v:-default}.csv
done
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "${TESTS:-space or pmg or scale or steady or dist}" \
  > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench_c4.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_c4.log
