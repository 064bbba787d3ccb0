#!/bin/bash
# ncu hot source lines of the panel kernel: cluster 8192 x 256 and grid (64 CTAs) 32768 x 256.  GPU box.
mkdir -p gpurun_out /tmp/prof
python tools/panel_once.py 8192 256 0 0 2 > /dev/null 2>&1 && \
timeout 300 ncu --set full --import-source on --clock-control none -k regex:panel_kernel -s 3 -c 1 -o /tmp/prof/pcl2 python tools/panel_once.py 8192 256 0 0 2 > gpurun_out/ph_ncu1.log 2>&1
timeout 200 python tools/ncu_source_hot.py /tmp/prof/pcl2.ncu-rep 45 > gpurun_out/ph_hot_cluster.txt 2>&1
python tools/panel_once.py 32768 256 64 0 1 > /dev/null 2>&1 && \
timeout 300 ncu --set full --import-source on --clock-control none -k regex:panel_kernel -s 3 -c 1 -o /tmp/prof/pgr2 python tools/panel_once.py 32768 256 64 0 1 > gpurun_out/ph_ncu2.log 2>&1
timeout 200 python tools/ncu_source_hot.py /tmp/prof/pgr2.ncu-rep 45 > gpurun_out/ph_hot_grid.txt 2>&1
