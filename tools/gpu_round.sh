mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c2_f64.csv python bench.py --steps 4 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"col_kernel|row" -c 4 -o gpurun_out/full_c2_f64 python tools/prof_step.py --iters 1 > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"col_kernel|row" -c 4 -o gpurun_out/full_c2_f32 python tools/prof_step.py --iters 1 --dtype float32 > gpurun_out/ncu_full32.log 2>&1; tail -1 gpurun_out/ncu_full32.log
