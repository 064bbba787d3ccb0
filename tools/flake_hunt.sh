# Repeat the bitwise panel / small-golden tests to look for rare races (exact mode is deterministic).
fails=0
for i in $(seq 1 25); do
  timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_getrf.py -q -x -k "panel_bitwise or small_golden or nan or zero_column" > /tmp/fh.log 2>&1 || { fails=$((fails+1)); tail -5 /tmp/fh.log; }
done
echo "flake hunt: $fails failing runs of 25"
