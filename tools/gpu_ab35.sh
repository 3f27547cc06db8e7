# rows-only permute at 6 CTAs/SM for Float64 (complex instances keep 4-5): f64 / c64 bench lines + parity
b() { python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 $2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['permute']['GB_s'], d['phase_ms'])"; }
b f64; b c64 "--dtype c64"
timeout 1300 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
