# round-2 final-tree checkpoint: c2 launch list + ncu full of the c2 kernels, ncu full of the c4 3D kernels
O=gpurun_out/r02n; mkdir -p $O
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c2_f64.csv python bench.py --steps 4 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"col_kernel|row" -c 4 -o $O/full_c2_f64 python tools/prof_step.py --iters 1 > $O/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"col_kernel|row" -c 3 -o $O/full_c4 python tools/prof_step.py --size 256 256 256 --dtype float32 --kinds dct_3d --iters 1 > $O/ncu_c4.log 2>&1
python tools/ncu_quick.py $O/full_c2_f64.ncu-rep > $O/full_c2_f64.txt 2>&1
python tools/ncu_quick.py $O/full_c4.ncu-rep > $O/full_c4.txt 2>&1
cat $O/full_c4.txt
