mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:"k_local_probe" -c 1 -f -o gpurun_out/r2_probe_new python tools/one_step.py 28 28 1.0 32 1 > gpurun_out/ncu_probe.log 2>&1
tail -3 gpurun_out/ncu_probe.log
