mkdir -p gpurun_out
ncu --set full --clock-control none --kernel-name-base demangled -k regex:"k_gemv_t|k_cgs_update_dot" -s 40 -c 2 -o gpurun_out/gemv1 -f \
    python tools/perf_probe.py --E 32 > gpurun_out/ncu_gemv1.log 2>&1
tail -2 gpurun_out/ncu_gemv1.log
