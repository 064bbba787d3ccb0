timeout 600 ncu --set full --import-source on --clock-control none -k regex:panel_kernel -s 3 -c 1 -o gpurun_out/panel2048_full python tools/panel_once.py 2048 256 > gpurun_out/p10_ncu.log 2>&1; tail -2 gpurun_out/p10_ncu.log
timeout 900 python tools/config_sweep.py gpurun_out/r03_configs.json > gpurun_out/r03_configs.log 2>&1; tail -20 gpurun_out/r03_configs.log
timeout 400 python bench.py > gpurun_out/p10_bench.json 2> gpurun_out/p10_bench.err; tail -1 gpurun_out/p10_bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['parity'], d['e2e']['value'])"
