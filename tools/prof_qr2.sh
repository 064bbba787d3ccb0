# QR evidence refresh: launch list of one n=8192 QR and a full capture of one cluster leaf (4096 rows).
python tools/qr_once.py 8192 256 1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qr_launches_8192_v2.csv \
      python tools/qr_once.py 8192 256 1 > gpurun_out/qr_ncu_list2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:qr_leaf_kernel --launch-skip 8 -c 1 \
    -o gpurun_out/qr_leaf_cluster_full -f python tools/qr_once.py 4096 256 0 > gpurun_out/qr_ncu_leaf2.log 2>&1
ls -la gpurun_out | grep qr_
