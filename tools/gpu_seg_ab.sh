# seg permute job size (TK_SEG_MAX, knob build _variants/libtk_knobs.so): 8192 (default) vs larger jobs
cd /root/repo
for i in 1 2; do
  for m in 8192 12288 16384 32768; do
    TK_LIB_PATH=_variants/libtk_knobs.so TK_SEG_MAX=$m timeout 300 python tools/bench_chains.py 2,3,5,6,7,8 > gpurun_out/seg_${m}_$i.jsonl 2>&1; echo "seg $m rc=$?"
  done
done
python - <<'PY'
import json
for i in (1,2):
  for m in (8192,12288,16384,32768):
    rows=[json.loads(l) for l in open(f"gpurun_out/seg_{m}_{i}.jsonl") if l.startswith("{")]
    print(m, i, [(r["cfg"], r["us_per_chain"]) for r in rows])
PY
