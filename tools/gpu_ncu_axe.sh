#!/bin/bash
# ncu --set full of k_axe<float> with the SASS source page (stall sampling per instruction)
T=${1:-r02ai}
bash tools/ncu_quick.sh "k_axe<.*float" ${T}_axe32 > /dev/null 2>&1
python tools/ncu_brief.py gpurun_out/${T}_axe32.ncu-rep > gpurun_out/${T}_axe32_ncu.txt 2>&1
ncu -i gpurun_out/${T}_axe32.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_axe32_src.csv 2>&1
ncu -i gpurun_out/${T}_axe32.ncu-rep --page source --csv --print-source cuda > gpurun_out/${T}_axe32_cuda.csv 2>&1
PROBE_ARGS="--solve 1" bash tools/ncu_quick.sh "k_cgs_update_norm" ${T}_norm > /dev/null 2>&1
python tools/ncu_brief.py gpurun_out/${T}_norm.ncu-rep > gpurun_out/${T}_norm_ncu.txt 2>&1
mkdir -p /tmp/k && mv gpurun_out/*.ncu-rep /tmp/k/
