timeout 900 python tools/emu_scaling.py --ranks 1,2,4,8 > gpurun_out/final_emu.log 2>&1; cut -c1-220 gpurun_out/final_emu.log
timeout 900 python tools/config_sweep.py gpurun_out/final_configs.json > gpurun_out/final_configs.log 2>&1; tail -16 gpurun_out/final_configs.log
