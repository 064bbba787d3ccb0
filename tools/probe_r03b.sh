set -x
for M in 2048 8192; do timeout 60 python tools/panel_prof.py $M 256 0 0 0 2; done > gpurun_out/p2_prof.log 2>&1
timeout 60 python tools/panel_prof.py 32768 256 0 0 0 1 >> gpurun_out/p2_prof.log 2>&1
timeout 60 python tools/panel_prof.py 8192 256 0 0 0 1 >> gpurun_out/p2_prof.log 2>&1
cat gpurun_out/p2_prof.log
timeout 120 python tools/panel_sweep.py --m 8192,4096,2048,1024 --kernel 2 --ctas 4,8,12,16 --reps 5 > gpurun_out/p2_sweep.log 2>&1
timeout 120 python tools/panel_sweep.py --m 32768,16384,8192 --kernel 1 --ctas 32,48,64,96,128 --reps 5 >> gpurun_out/p2_sweep.log 2>&1
timeout 120 python tools/panel_sweep.py --m 4096,2048,1024 --w 128 --kernel 1,2 --reps 5 >> gpurun_out/p2_sweep.log 2>&1
grep median gpurun_out/p2_sweep.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv python tools/panel_once.py 32768 256 0 0 3 > gpurun_out/p2_rec_launches.csv 2> gpurun_out/p2_rec_launches.err
tail -2 gpurun_out/p2_rec_launches.err
timeout 900 python tools/emu_scaling.py --ranks 1,8 --b 128 > gpurun_out/p2_emu.log 2>&1
PFLU_GRID_ROWS=4096 timeout 600 python tools/emu_scaling.py --ranks 8 >> gpurun_out/p2_emu.log 2>&1
PFLU_GRID_ROWS=100000 timeout 600 python tools/emu_scaling.py --ranks 8 >> gpurun_out/p2_emu.log 2>&1
cat gpurun_out/p2_emu.log
