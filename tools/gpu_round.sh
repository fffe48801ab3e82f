mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"col2" -c 2 -o gpurun_out/col2 python tools/prof_step.py --iters 1 > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
