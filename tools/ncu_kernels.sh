#!/bin/bash
# usage: tools/ncu_kernels.sh <regex> <count> <outname> [probe args]
mkdir -p gpurun_out
python tools/perf_probe.py --E 32 --solve ${SOLVE:-0} > gpurun_out/probe_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$1" -s 3 -c "$2" -o gpurun_out/"$3" -f \
    python tools/perf_probe.py --E 32 --solve ${SOLVE:-0} > gpurun_out/ncu_$3.log 2>&1
tail -3 gpurun_out/ncu_$3.log
