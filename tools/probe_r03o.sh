timeout 900 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/p14_tests.log 2>&1; tail -2 gpurun_out/p14_tests.log
timeout 600 python bench.py --dist --steps 2 --warmup 3 --e2e-steps 2 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['e2e'])"
