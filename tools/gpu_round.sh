mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 400 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -2 gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json
for wl in c1 c3 c4 c5; do timeout 400 python bench.py --workload $wl --steps 50 > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err; tail -2 gpurun_out/bench_$wl.err; cat gpurun_out/bench_$wl.json; done
timeout 300 python bench.py --dtype float32 --no-cpu > gpurun_out/bench_c2_f32.json 2>&1; cat gpurun_out/bench_c2_f32.json
