python -m pytest tests/test_gpu_edge.py -x -q -k bulk > gpurun_out/r2l_pytest.log 2>&1; echo "bulk pytest rc=$?"; tail -1 gpurun_out/r2l_pytest.log
for v in default b4 b3nb3 nobulk; do
  case $v in default) E="";; nobulk) E="TK_LIB_PATH=_variants/libtk_knobs.so TK_NO_BULK=1";; *) E="TK_LIB_PATH=_variants/libtk_$v.so";; esac
  env $E python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-chains > gpurun_out/r2l_bench_$v.json 2> gpurun_out/r2l_bench_$v.err; echo "bench $v rc=$?"
  python -c "
import json
d=json.load(open('gpurun_out/r2l_bench_$v.json'))
print('$v', d['value'], d['phase_ms'], d['roofline_permute']['frac'])
"
done
