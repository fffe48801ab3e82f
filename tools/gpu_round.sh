timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for s in "6000 6000" "5000 4100" "1000 1000"; do timeout 120 python tools/stage_time.py --dtype float64 --size $s --kinds dct_2d 2>&1 | tail -1; done
