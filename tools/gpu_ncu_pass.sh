#!/bin/bash
# ncu --set full of the pMG transfer passes (x prolong / x restrict / y restrict) at c4
T=${1:-r02w}
export PROBE_ARGS="--solve 1"
bash tools/ncu_quick.sh "k_pass_x<.bool.0, .int.7" ${T}_pr00 > /dev/null 2>&1
bash tools/ncu_quick.sh "k_pass_x<.bool.1, .int.7" ${T}_pp10 > /dev/null 2>&1
bash tools/ncu_quick.sh "k_pass_ycol<.bool.1" ${T}_pr01 > /dev/null 2>&1
for k in pr00 pp10 pr01; do python tools/ncu_brief.py gpurun_out/${T}_$k.ncu-rep > gpurun_out/${T}_${k}_ncu.txt 2>&1;
 ncu -i gpurun_out/${T}_$k.ncu-rep --page details > gpurun_out/${T}_${k}_details.txt 2>&1; ncu -i gpurun_out/${T}_$k.ncu-rep --page source --csv > gpurun_out/${T}_${k}_src.csv 2>&1; done
mkdir -p /tmp/k && mv gpurun_out/*.ncu-rep /tmp/k/
