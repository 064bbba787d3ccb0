timeout 900 python tools/emu_scaling.py --ranks 1,2,4,8 > gpurun_out/p12_emu_default.log 2>&1; cat gpurun_out/p12_emu_default.log | cut -c1-200
PFLU_GRID_ROWS=1000000000 timeout 900 python tools/emu_scaling.py --ranks 2,4,8 > gpurun_out/p12_emu_cluster.log 2>&1; cat gpurun_out/p12_emu_cluster.log | cut -c1-200
timeout 600 python bench.py --dist --steps 2 --warmup 3 --e2e-steps 0 --no-cpu 2>/dev/null | tail -1 | cut -c1-200
