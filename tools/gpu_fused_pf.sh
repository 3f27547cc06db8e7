# fused MPO pair: per-tree loads (default) vs next-tree prefetch (-DTK_FUSED_PREFETCH=1, _variants/libtk_pf.so)
cd /root/repo
TK_LIB_PATH=_variants/libtk_pf.so timeout 900 python -m pytest tests/test_gpu_fused.py -q -x > gpurun_out/pf_pytest.log 2>&1; echo "pytest pf rc=$?"; tail -1 gpurun_out/pf_pytest.log
for i in 1 2 3; do
  timeout 300 python tools/bench_chains.py 2,3,8 > gpurun_out/pf_base_$i.jsonl 2>&1; echo "base rc=$?"
  TK_LIB_PATH=_variants/libtk_pf.so timeout 300 python tools/bench_chains.py 2,3,8 > gpurun_out/pf_pf_$i.jsonl 2>&1; echo "pf rc=$?"
done
python - <<'PY'
import json
for tag in ("base_1","pf_1","base_2","pf_2","base_3","pf_3"):
    rows=[json.loads(l) for l in open(f"gpurun_out/pf_{tag}.jsonl") if l.startswith("{")]
    print(tag, [(r["cfg"], r["us_per_chain"]) for r in rows])
PY
