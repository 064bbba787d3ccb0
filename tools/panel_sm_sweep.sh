#!/bin/bash
# Panel-cluster sizing vs the concurrent trailing GEMM: C2 / C3 / C4 device-resident times for
# PFLU_CL_MINROWS (rows per panel CTA at least) and PFLU_CLUSTER (max CTAs).  GPU box.
for cfg in "PFLU_CL_MINROWS=128" "PFLU_CL_MINROWS=512" "PFLU_CL_MINROWS=1024" "PFLU_CL_MINROWS=2048" "PFLU_CLUSTER=8" "PFLU_CLUSTER=12"; do
  echo "== $cfg"
  env PROBE_DYNAMIC_ONLY=1 $cfg timeout 300 python tools/malleable_probe.py 8192 16384 32768 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['n'], d['dynamic_ms'])"
done
