#!/bin/bash
# Runs on the GPU box: plain bench, launch list, and full ncu captures of the top kernels.
set -x
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 > gpurun_out/bench.log 2>&1 || exit 1
tail -1 gpurun_out/bench.log
if [ "${NCU:-1}" = "1" ]; then
  python tools/perf_probe.py --E 32 --solve 1 > gpurun_out/probe_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:'k_axp|k_ras' -s 12 -c 6 \
      -o gpurun_out/prof_top -f python tools/perf_probe.py --E 32 --solve 1 > gpurun_out/ncu_full.log 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none -s 2500 -c 3000 --csv \
      --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
fi
exit 0
