for lib in lib lib_noxs; do
  export LD_LIBRARY_PATH=$PWD/paper_2110_01172_b200/$lib
  echo "=== $lib"
  python tools/stage_time.py --reps 40; python tools/stage_time.py --dtype float32 --reps 40
  python tools/trace_col.py 4096 float64 | head -12
  python bench.py --no-cpu --steps 100 --warmup 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['ms_per_step'], d['roofline']['all_kernels'])"
  python bench.py --no-cpu --steps 100 --warmup 10 --dtype float32 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench32', d['ms_per_step'], d['roofline']['all_kernels'])"
done
