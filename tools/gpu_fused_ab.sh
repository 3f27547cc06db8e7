# fused MPO-pair kernel variants: parity + A/B (old = previous build, new = program staged in shared memory,
# hoist = the same with all inputs hoisted)
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_ncon.py -q -x > gpurun_out/fab_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/fab_pytest.log
TK_LIB_PATH=_variants/libtk_hoist.so timeout 900 python -m pytest tests/test_gpu_fused.py -q -x > gpurun_out/fab_pytest_hoist.log 2>&1; echo "pytest hoist rc=$?"; tail -1 gpurun_out/fab_pytest_hoist.log
for i in 1 2; do
  TK_LIB_PATH=_variants/libtk_old.so timeout 300 python tools/bench_chains.py 2,3,8 > gpurun_out/fab_old_$i.jsonl 2>&1; echo "old rc=$?"
  timeout 300 python tools/bench_chains.py 2,3,8 > gpurun_out/fab_new_$i.jsonl 2>&1; echo "new rc=$?"
  TK_LIB_PATH=_variants/libtk_hoist.so timeout 300 python tools/bench_chains.py 2,3,8 > gpurun_out/fab_hoist_$i.jsonl 2>&1; echo "hoist rc=$?"
done
python - <<'PY'
import json
for tag in ("old_1","new_1","hoist_1","old_2","new_2","hoist_2"):
    rows=[json.loads(l) for l in open(f"gpurun_out/fab_{tag}.jsonl") if l.startswith("{")]
    print(tag, [(r["cfg"], r["us_per_chain"], r.get("us_per_chain_pairwise")) for r in rows])
PY
timeout 300 ncu -k regex:fused_pair -c 1 --set full --import-source on --clock-control none -o gpurun_out/fused_new python tools/prof_chain.py 3 > gpurun_out/fab_ncu.log 2>&1; echo "ncu rc=$?"
