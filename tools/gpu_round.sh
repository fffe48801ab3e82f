mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for s in "1000 1000" "3000 2000" "1536 1536" "4099 256" "100 60 90"; do timeout 120 python tools/stage_time.py --dtype float64 --size $s --kinds dct_2d 2>&1 | tail -1; done
