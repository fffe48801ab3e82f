# graph-mode bench lines for every config (+ eager c1 for comparison)
O=gpurun_out/r02h; mkdir -p $O
for c in c1 c2 c3 c4 c5 cz; do timeout 400 python bench.py --workload $c --no-cpu > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"; done
timeout 300 python bench.py --workload c1 --no-cpu --eager > $O/bench_c1_eager.json 2> $O/bench_c1_eager.err
timeout 300 python bench.py --workload c2 --dtype float32 --no-cpu > $O/bench_c2_f32.json 2> $O/bench_c2_f32.err
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r02h/bench_*.json')):
    try: d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e: print(f, 'ERR', e); continue
    r=d['roofline']; cf=d.get('cufft',{})
    print(f.split('/')[-1], d['ms_per_step'], d['value'], r['frac'], [(k['kernel'],round(k['ms']*1e3,1)) for k in r['all_kernels']], d['measurement'].get('launch','')[:40], {k:v for k,v in cf.items() if k.endswith('_ms') or 'over' in k})
PY
