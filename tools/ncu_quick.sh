#!/bin/bash
# usage: tools/ncu_quick.sh <kernel regex> <outname> [lib variant]  (one --set full capture of the E=32^3 probe)
mkdir -p gpurun_out
[ -n "$3" ] && export SEMLAB_LIB=$3
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$1" -s 3 -c 1 -o gpurun_out/"$2" -f \
    python tools/perf_probe.py --E 32 ${PROBE_ARGS:---solve 0} > gpurun_out/ncu_$2.log 2>&1
tail -2 gpurun_out/ncu_$2.log
