PFLU_LSWAP_TW=8 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k "laswp" 2>&1 | tail -1
for B in 8 16 8 16; do PFLU_LSWAP_TW=$B timeout 300 python bench.py --e2e-steps 0 --no-cpu --no-check 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('tw=$B', round(d['ms_per_step'],2), round(d['roofline']['achieved'],3))"; done
