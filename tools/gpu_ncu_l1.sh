#!/bin/bash
# ncu --set full of the p=3 level kernels (RAS P=6 step mode, Ax, gather) at c4
T=${1:-r02ae}
export PROBE_ARGS="--solve 1"
bash tools/ncu_quick.sh "k_ras<.int.6, float, .int.2" ${T}_ras6 > /dev/null 2>&1
bash tools/ncu_quick.sh "k_ax<.int.4" ${T}_ax4 > /dev/null 2>&1
bash tools/ncu_quick.sh "k_gather_epi<.int.4" ${T}_gat4 > /dev/null 2>&1
for k in ras6 ax4 gat4; do python tools/ncu_brief.py gpurun_out/${T}_$k.ncu-rep > gpurun_out/${T}_${k}_ncu.txt 2>&1;
 ncu -i gpurun_out/${T}_$k.ncu-rep --page source --csv > gpurun_out/${T}_${k}_src.csv 2>&1; done
mkdir -p /tmp/k && mv gpurun_out/*.ncu-rep /tmp/k/
