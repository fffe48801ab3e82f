# Round-end measurement script (run under gpurun from the repo root)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 400 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 400 python bench.py --dtype float32 > gpurun_out/bench_c2_f32.json 2> gpurun_out/bench_c2_f32.err
for wl in c1 c3 c4 c5 cz; do timeout 500 python bench.py --workload $wl --steps 50 > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c2_f64.csv python bench.py --steps 4 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"col_kernel|row" -c 4 -o gpurun_out/full_c2_f64 python tools/prof_step.py --iters 1 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"col_kernel|row" -c 4 -o gpurun_out/full_c2_f32 python tools/prof_step.py --iters 1 --dtype float32 > gpurun_out/ncu_full32.log 2>&1
ls gpurun_out
