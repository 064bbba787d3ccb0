timeout 900 python -m pytest tests/test_gpu_getrf.py -q -x -k "not c5 and not c4" 2>&1 | tail -1
for i in 1 2; do timeout 200 python bench.py --steps 1 --warmup 3 --e2e-steps 4 --no-cpu --no-check 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('e2e', d['e2e']['ms_per_step'], d['e2e']['value'])"; done
