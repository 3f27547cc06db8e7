set -x
python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r2b_bench_tma.json 2> gpurun_out/r2b_bench_tma.err; echo "bench rc=$?"
tail -3 gpurun_out/r2b_bench_tma.err
python -c "
import json
d=json.load(open('gpurun_out/r2b_bench_tma.json'))
print(d['value'], d['roofline'], d['phase_ms'], d['gpu_launches'])
for k,v in (d.get('chains') or {}).items(): print(k, v)
"
