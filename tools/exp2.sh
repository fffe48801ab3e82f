timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python tools/stage_time.py; python tools/stage_time.py --dtype float32
python tools/stage_time.py --size 4096 2048 --kinds dct_2d,idct_2d,idct_idxst_2d
