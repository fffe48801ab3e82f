timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for r in 1 0; do SDCT_ROWP=$r python tools/stage_time.py --reps 40; done
SDCT_ROWP=1 python tools/stage_time.py --kinds idct_idxst_2d,idxst_idct_2d --reps 20
python bench.py --no-cpu --steps 100 --warmup 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['ms_per_step'], d['roofline']['frac'], d['roofline']['all_kernels'], d['parity'])"
