#!/bin/bash
# usage: tools/ncu_times.sh <kernel regex> <out.csv>  -- per-launch durations over the E=32^3 probe solve
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$1" --csv --log-file gpurun_out/$2 \
    python tools/perf_probe.py --E 32 > /dev/null 2>&1
