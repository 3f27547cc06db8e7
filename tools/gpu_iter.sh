python tools/bench_configs.py --cfgs 2,3,5 --reps 30 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['permute'])"
python tools/prof_chain.py 3 2 >/dev/null && ncu --set full --clock-control none --import-source on -k regex:"permute_kernel" -s 1 -c 1 -o gpurun_out/prof_cfg3_perm python tools/prof_chain.py 3 1 > gpurun_out/ncu_cfg3p.log 2>&1; echo ncu=$?
