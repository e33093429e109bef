#!/bin/bash
# One --set full capture each of the two roofline kernels exactly as bench.py times them:
# the FP64 Krylov Ax (k_axw<EWrite, double>) and the plain FP32 RAS apply (k_rasw<10, float, 0>),
# at the bench workload (perf_probe E=32^3). Output: gpurun_out/roof_<R>.ncu-rep
R=${ROUND:-r01}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"k_axw|k_rasw" -s 3 -c 2 -o gpurun_out/roof_$R -f \
    python tools/perf_probe.py --E 32 --solve 0 > gpurun_out/ncu_roof_$R.log 2>&1
tail -1 gpurun_out/ncu_roof_$R.log
