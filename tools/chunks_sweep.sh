#!/bin/bash
# Trailing column-chunk streams (PFLU_CHUNKS) with the WS GEMM: C3 / C4 device-resident times.
for ch in 1 2 3 4 6; do
  echo "== PFLU_CHUNKS=$ch"
  PROBE_DYNAMIC_ONLY=1 PFLU_CHUNKS=$ch timeout 300 python tools/malleable_probe.py 16384 32768 2>&1 | grep "^{"
done
