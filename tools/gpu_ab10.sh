# A/B: double-buffered box kernel (TK_BOX=1) vs rows path on the cfg4 permutes; parity with TK_BOX=1
python tools/perm_bench.py 384 2>&1 | tail -3
TK_BOX=1 python tools/perm_bench.py 384 2>&1 | tail -3
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rows', d['value'], d['permute'])"
TK_BOX=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('box', d['value'], d['permute'])"
TK_BOX=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cfg4 or large or permute_random" 2>&1 | tail -2
