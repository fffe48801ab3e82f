mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for f in 0 1; do for m in 0 1; do SDCT_DEV_FLAGS=$f SDCT_ROW2_MODE=$m timeout 120 python tools/stage_time.py --dtype float64; done; done
SDCT_ROW2_MODE=0 timeout 120 python tools/stage_time.py --dtype float32
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"row2" -c 2 -o gpurun_out/row2_m0 python tools/prof_step.py --iters 1 > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
