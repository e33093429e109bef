#!/bin/bash
# 1-GPU profiling batch: Ax variant A/B, ncu --set full of the roofline kernels (traffic), tests, bench.
T=${1:-prof}
mkdir -p gpurun_out
for v in ""; do
  if [ -z "$v" ]; then lib=libsemlab_b200.so; else lib=libsemlab_b200_$v.so; fi
  SEMLAB_LIB=$lib timeout 300 python tools/perf_probe.py --solve 1 > gpurun_out/${T}_probe_${v:-default}.log 2>&1
done
bash tools/ncu_quick.sh "k_axe.*double" ${T}_axe64 > /dev/null 2>&1
bash tools/ncu_quick.sh "k_axe.*float" ${T}_axe32 > /dev/null 2>&1
bash tools/ncu_quick.sh "k_face_epi7" ${T}_face > /dev/null 2>&1
bash tools/ncu_quick.sh "k_rasw" ${T}_rasw > /dev/null 2>&1
for k in axe64 axe32 face rasw; do python tools/ncu_brief.py gpurun_out/${T}_$k.ncu-rep > gpurun_out/${T}_${k}_ncu.txt 2>&1; done
python tools/traffic_summary.py gpurun_out/${T}_axe64.ncu-rep gpurun_out/${T}_axe32.ncu-rep gpurun_out/${T}_face.ncu-rep \
  gpurun_out/${T}_rasw.ncu-rep gpurun_out/${T}_latest_ncu_summary.json > /dev/null 2>&1
mkdir -p /tmp/ncu_keep && mv gpurun_out/${T}_*.ncu-rep /tmp/ncu_keep/  # reports stay on the box (64 MiB pull limit)
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench_c4.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_c4.log
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 > gpurun_out/${T}_bench_c1.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench_c1.log
