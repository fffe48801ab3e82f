# round-2 checkpoint 2: bench lines for all configs + launch list + ncu full of c2 fp64
mkdir -p gpurun_out/r02f
O=gpurun_out/r02f
timeout 400 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 400 python bench.py --dtype float32 --no-cpu > $O/bench_c2_f32.json 2> $O/bench_c2_f32.err
for wl in c1 c3 c4 c5 cz; do timeout 500 python bench.py --workload $wl --steps 50 > $O/bench_$wl.json 2> $O/bench_$wl.err; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c2_f64.csv python bench.py --steps 4 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"col_kernel|row" -c 4 -o $O/full_c2_f64 python tools/prof_step.py --iters 1 > $O/ncu_full.log 2>&1
ls $O
