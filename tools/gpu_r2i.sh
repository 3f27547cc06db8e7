timeout 600 python tools/bench_configs.py --cfgs 2,3,7 --reps 30 --phases > gpurun_out/r2i_configs.jsonl 2> gpurun_out/r2i_configs.err; echo "configs rc=$?"
python -c "
import json
for l in open('gpurun_out/r2i_configs.jsonl'):
    d=json.loads(l); print(d['cfg'], d['us_per_chain_graph'], d['launches'], d.get('phase_us_per_step'))
"
python tools/prof_chain.py 3 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r2i_cfg3_launches.csv python tools/prof_chain.py 3 > /dev/null 2>&1; echo "ncu rc=$?"
python -c "
import csv
rows=list(csv.reader(open('gpurun_out/r2i_cfg3_launches.csv')))
h=rows[0]
for r in rows[1:40]:
    d=dict(zip(h,r))
    if d.get('Metric Name')=='gpu__time_duration.sum': print(d['Kernel Name'][:60], d['Grid Size'], d['Metric Value'])
"
