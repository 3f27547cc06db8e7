for v in default split22 split21 split23 bk32 st2; do
  case $v in default) E="";; split2*) E="TK_LIB_PATH=_variants/libtk_knobs.so TK_SPLIT_LOG2=${v#split}";; *) E="TK_LIB_PATH=_variants/libtk_$v.so";; esac
  echo "== $v"; env $E timeout 300 python tools/bench_configs.py --cfgs 2,3,7 --reps 30 --phases 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], d['launches'], d.get('phase_us_per_step'))
"
done
