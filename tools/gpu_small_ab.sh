# A/B of the 64 x 64 DMMA tile (gemm_tile): default build against _variants/libtk_head.so (the previous
# commit, tools/build_variant.sh head ""): parity of the default build, then the chains (bench_chains.py:
# tk_ncon and pairwise, CUDA graphs, L2 flushed) alternating, then per-phase times of the configs.
set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py tests/test_gpu_fused.py tests/test_gpu_ncon.py -m gpu -q -x > gpurun_out/small_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/small_pytest.log
for r in 1 2; do
  python tools/bench_chains.py 2,3,5,6,7,8 > gpurun_out/small_new_$r.jsonl 2> gpurun_out/small_new_$r.err; echo "new rc=$?"
  TK_LIB_PATH=_variants/libtk_head.so python tools/bench_chains.py 2,3,5,6,7,8 > gpurun_out/small_old_$r.jsonl 2> gpurun_out/small_old_$r.err; echo "old rc=$?"
done
python tools/bench_configs.py --reps 30 --phases > gpurun_out/small_new_phases.jsonl 2>/dev/null
TK_LIB_PATH=_variants/libtk_head.so python tools/bench_configs.py --reps 30 --phases > gpurun_out/small_old_phases.jsonl 2>/dev/null
python - <<'PY'
import json
for n in ("new_1", "old_1", "new_2", "old_2"):
    rows = [json.loads(l) for l in open(f"gpurun_out/small_{n}.jsonl") if l.startswith("{")]
    print(n, {r["cfg"]: (r["us_per_chain"], r["us_per_chain_pairwise"]) for r in rows})
for n in ("new", "old"):
    rows = [json.loads(l) for l in open(f"gpurun_out/small_{n}_phases.jsonl") if l.startswith("{")]
    print(n, {r["cfg"]: (r["us_per_chain_graph"], [p[2] for p in r["phase_us_per_step"]]) for r in rows})
PY
