# round-2 probe: column-pass phase traces (4096^2, 1024^2 fp64), c1 latency probe, ncu full of c1 kernels
O=gpurun_out/r02g; mkdir -p $O
timeout 120 python tools/trace_col.py 4096 float64 > $O/trace4096.txt 2>&1
timeout 300 bash tools/c1_probe.sh > $O/c1_probe.txt 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"col_kernel|row" -c 4 -o $O/full_c1 python tools/prof_step.py --size 1024 1024 --iters 1 > $O/ncu_c1.log 2>&1
python tools/ncu_quick.py $O/full_c1.ncu-rep > $O/full_c1.txt 2>&1
