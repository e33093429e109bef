#!/bin/bash
# ncu --set full of the fused Chebyshev-RAS step (k_rasw mode 2) with the SASS source page
T=${1:-r02ao}
export PROBE_ARGS="--solve 1"
bash tools/ncu_quick.sh "k_rasw<.int.10, float, .int.2" ${T}_rasw2 > /dev/null 2>&1
python tools/ncu_brief.py gpurun_out/${T}_rasw2.ncu-rep > gpurun_out/${T}_rasw2_ncu.txt 2>&1
ncu -i gpurun_out/${T}_rasw2.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_rasw2_src.csv 2>&1
mkdir -p /tmp/k && mv gpurun_out/*.ncu-rep /tmp/k/
