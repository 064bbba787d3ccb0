run() { echo "== $*"; env "$@" timeout 600 python tools/emu_scaling.py --ranks 1,8 2>&1 | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['P'], round(d['model_ms'],1), 'eff', round(d['model_efficiency'] or 0,3), 'pf', round(d['sum_pf_ms'],1), 'tul', round(d['sum_tul_ms'],1))"; }
run X=0
run PFLU_PANEL_CAP=96
run PFLU_PANEL_CAP=128
run PFLU_GRID_ROWS=4096
run PFLU_GRID_ROWS=4096 PFLU_PANEL_CAP=48
run PFLU_GRID_ROWS=2048 PFLU_PANEL_CAP=96
