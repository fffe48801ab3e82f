mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 400 python bench.py --workload c3 --steps 50 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -3 gpurun_out/bench_c3.err; cat gpurun_out/bench_c3.json
for dt in float64 float32; do timeout 120 python tools/stage_time.py --dtype $dt --size 256 256 256 --kinds dct_3d,idct_3d; done
