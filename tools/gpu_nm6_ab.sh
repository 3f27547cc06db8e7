# fused MPO pair: NM = 6 coefficient rows for K, N <= 6 (cfg3) vs the previous build (_variants/libtk_head.so)
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_ncon.py -q -x > gpurun_out/nm6_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/nm6_pytest.log
for i in 1 2 3; do
  TK_LIB_PATH=_variants/libtk_head.so timeout 300 python tools/bench_chains.py 3,7 > gpurun_out/nm6_head_$i.jsonl 2>&1; echo "head rc=$?"
  timeout 300 python tools/bench_chains.py 3,7 > gpurun_out/nm6_new_$i.jsonl 2>&1; echo "new rc=$?"
done
python - <<'PY'
import json
for i in (1,2,3):
  for tag in ("head","new"):
    rows=[json.loads(l) for l in open(f"gpurun_out/nm6_{tag}_{i}.jsonl") if l.startswith("{")]
    print(tag, i, [(r["cfg"], r["us_per_chain"]) for r in rows])
PY
timeout 300 ncu -k regex:fused_pair -c 1 --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none python tools/prof_chain.py 3 2>&1 | grep -E "fused|duration|inst_exec|warps_active" | head -8
