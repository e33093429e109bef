#!/bin/bash
# 1-GPU check after a kernel change: probe, per-launch times of the transfer / Ax kernels, the face
# kernel's ncu brief, the space/pMG parity tests and the c4 bench.
T=${1:-q}
mkdir -p gpurun_out
timeout 300 python tools/perf_probe.py --solve 1 > gpurun_out/${T}_probe.log 2>&1
timeout 300 bash tools/ncu_times.sh "k_pass|k_face|k_axe|k_rasw" ${T}_times.csv
bash tools/ncu_quick.sh "k_face_epi7" ${T}_face > /dev/null 2>&1
python tools/ncu_brief.py gpurun_out/${T}_face.ncu-rep > gpurun_out/${T}_face_ncu.txt 2>&1
mkdir -p /tmp/ncu_keep && mv gpurun_out/${T}_*.ncu-rep /tmp/ncu_keep/
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "space or pmg or scale or steady" \
  > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench_c4.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_c4.log
