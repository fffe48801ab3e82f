# round-2 final bench lines (graph-replayed timed steps) for every config, the reference arm, smoke, acceptance
O=gpurun_out/r02o; mkdir -p $O
for c in c2 c1 c3 c4 c5 cz; do timeout 400 python bench.py --workload $c > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"; done
timeout 300 python bench.py --workload c2 --dtype float32 --no-cpu > $O/bench_c2_f32.json 2> $O/bench_c2_f32.err
timeout 400 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r02o/bench_*.json')):
    try: d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e: print(f, 'ERR', e); continue
    r=d.get('roofline') or {}; cf=d.get('cufft',{}) or {}
    print(f.split('/')[-1], d.get('ms_per_step'), d.get('value'), r.get('frac'), [(k['kernel'],round(k['ms']*1e3,1)) for k in r.get('all_kernels',[])], (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'), {k:v for k,v in cf.items() if 'over' in k}, d.get('clocks'))
PY
