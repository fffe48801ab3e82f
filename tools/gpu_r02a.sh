# round-2 checkpoint: tests, smoke, acceptance, c2 bench lines, launch list, ncu full of c2 fp64
mkdir -p gpurun_out/r02a
O=gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q -x > $O/gpu_tests.log 2>&1; tail -3 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 tests/cpp/bin/acceptance_dropin > $O/acceptance.log 2>&1; tail -2 $O/acceptance.log
timeout 400 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; cat $O/bench_c2.json
timeout 400 python bench.py --dtype float32 --no-cpu > $O/bench_c2_f32.json 2> $O/bench_c2_f32.err
timeout 300 python tools/stage_time.py > $O/stage_c2_f64.txt 2>&1
timeout 300 python tools/stage_time.py --dtype float32 > $O/stage_c2_f32.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c2_f64.csv python bench.py --steps 4 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"col_kernel|row" -c 4 -o $O/full_c2_f64 python tools/prof_step.py --iters 1 > $O/ncu_full.log 2>&1
ls $O
