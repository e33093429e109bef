#!/bin/bash
# Runs on the GPU box (one GPU): the default bench line, the ncu launch list of the bench command
# (per-launch times, cold cache, serialised) and one --set full capture of the top kernels.
# Outputs land in gpurun_out/; tools/profile_summary.py turns them into profiles/<round>_*.
R=${ROUND:-r01}
set -x
mkdir -p gpurun_out
if [ "${FULL_ONLY:-0}" = "0" ]; then
  python bench.py > gpurun_out/bench_$R.log 2>&1 || exit 1
  tail -1 gpurun_out/bench_$R.log
  ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
      --log-file gpurun_out/launches_$R.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
      > gpurun_out/ncu_launches_$R.log 2>&1
fi
if [ "${NCU:-1}" = "1" ]; then
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:"${KREGEX:-k_axw|k_rasw|k_pass|k_cgs_update_dot|k_gemv_t}" -s ${SKIP:-60} -c ${COUNT:-16} \
      --nvtx --nvtx-include "timed/" -o gpurun_out/full_$R${TAG:-} -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_$R${TAG:-}.log 2>&1
fi
exit 0
