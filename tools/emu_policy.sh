for GR in 16384 24576; do PFLU_EMU_GRID_RANKS=2 PFLU_GRID_ROWS=$GR timeout 900 python tools/emu_scaling.py --ranks 2,4,8 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('grid_rows=$GR', d['P'], round(d['model_ms'],1), round(d['sum_pf_ms'],1))"; done
