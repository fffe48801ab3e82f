for rep in 1 2; do for v in 0 1; do
SDCT_ROWINV_REV=$v timeout 300 python bench.py --workload c2 --no-cpu --steps 100 > gpurun_out/ab_c2_$v.json 2>/dev/null
SDCT_ROWINV_REV=$v timeout 300 python bench.py --workload c2 --dtype float32 --no-cpu --steps 100 > gpurun_out/ab_c2f_$v.json 2>/dev/null
SDCT_ROWINV_REV=$v timeout 300 python bench.py --workload c3 --no-cpu --steps 100 > gpurun_out/ab_c3_$v.json 2>/dev/null
python - <<PY
import json
for c in ("c2","c2f","c3"):
    d=json.loads(open(f"gpurun_out/ab_{c}_$v.json").read().strip().splitlines()[-1])
    print("rev=$v", c, d["ms_per_step"], [(k["kernel"], round(k["ms"]*1e3,1)) for k in d["roofline"]["all_kernels"]], d["parity"])
PY
done; done
SDCT_ROWINV_REV=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "idct or force or compress or golden" 2>&1 | tail -2
