python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py tests/test_gpu_ncon.py tests/test_gpu_capture.py -x -q > gpurun_out/r2o_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2o_pytest.log
for v in default notma; do
  case $v in default) E="";; notma) E="TK_LIB_PATH=_variants/libtk_knobs.so TK_NO_TMA=1";; esac
  echo "== $v"; env $E timeout 300 python tools/bench_configs.py --cfgs 1,2,3,5,6,7,8 --reps 30 --phases 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], d['launches'], d.get('phase_us_per_step'))
"
done
