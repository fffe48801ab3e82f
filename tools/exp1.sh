for m in 0 1 2; do SDCT_ROW2_MODE=$m python tools/stage_time.py; SDCT_ROW2_MODE=$m python tools/stage_time.py --dtype float32; done
SDCT_ROW2_MODE=0 python tools/stage_time.py --size 2048 2048
SDCT_ROW2_MODE=1 python tools/stage_time.py --size 2048 2048
SDCT_ROW2_MODE=2 python tools/stage_time.py --size 2048 2048
