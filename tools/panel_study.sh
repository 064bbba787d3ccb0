#!/bin/bash
# Panel kernel study (GPU box): timing sweep, per-phase clocks, ncu hot source lines of the cluster
# kernel at 8192 x 256 and the grid kernel at 32768 x 256.
mkdir -p gpurun_out /tmp/prof
timeout 300 python tools/panel_sweep.py --m 32768,16384,8192,4096,2048,1024 --kernel 1,2 --w 256 > gpurun_out/ps_sweep256.log 2>&1
timeout 300 python tools/panel_sweep.py --m 8192,4096,2048,1024 --kernel 1,2 --w 128 > gpurun_out/ps_sweep128.log 2>&1
for args in "2048 128 0 0 0 2" "8192 256 0 0 0 2" "32768 256 64 0 0 1"; do
  echo "== $args"; timeout 120 python tools/panel_prof.py $args
done > gpurun_out/ps_prof.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:panel_kernel -s 3 -c 1 -o /tmp/prof/pcl python tools/panel_once.py 8192 256 0 0 2 > gpurun_out/ps_ncu1.log 2>&1
timeout 200 python tools/ncu_source_hot.py /tmp/prof/pcl.ncu-rep 60 > gpurun_out/ps_hot_cluster.txt 2>&1
ncu -i /tmp/prof/pcl.ncu-rep --page raw --csv > gpurun_out/ps_cluster_raw.csv 2>/dev/null
