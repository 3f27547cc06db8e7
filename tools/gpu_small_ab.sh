# small-tile GEMM: CTA-barrier pipeline (default) vs the mbarrier-pipelined tile (smb4: 4 stages, PD 2;
# smb5: 5 stages, PD 3) on the DMRG chains; parity of the variant and of the default build
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_ncon.py -q -x > gpurun_out/sab_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/sab_pytest.log
TK_LIB_PATH=_variants/libtk_smb4.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x > gpurun_out/sab_pytest_smb4.log 2>&1; echo "pytest smb4 rc=$?"; tail -1 gpurun_out/sab_pytest_smb4.log
for i in 1 2; do
  timeout 300 python tools/bench_chains.py 2,3,7,8 > gpurun_out/sab_base_$i.jsonl 2>&1; echo "base rc=$?"
  TK_LIB_PATH=_variants/libtk_smb4.so timeout 300 python tools/bench_chains.py 2,3,7,8 > gpurun_out/sab_smb4_$i.jsonl 2>&1; echo "smb4 rc=$?"
  TK_LIB_PATH=_variants/libtk_smb5.so timeout 300 python tools/bench_chains.py 2,3,7,8 > gpurun_out/sab_smb5_$i.jsonl 2>&1; echo "smb5 rc=$?"
done
python - <<'PY'
import json
for tag in ("base_1","smb4_1","smb5_1","base_2","smb4_2","smb5_2"):
    rows=[json.loads(l) for l in open(f"gpurun_out/sab_{tag}.jsonl") if l.startswith("{")]
    print(tag, [(r["cfg"], r["us_per_chain"], r.get("us_per_chain_pairwise")) for r in rows])
PY
