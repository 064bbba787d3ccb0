"""Print how many 16-CTA panel clusters the device holds at once (cudaOccupancyMaxActiveClusters is
queried inside libpflu; here: time the multi-cluster panel for a few cluster counts)."""
import os
import subprocess
import sys

for maxcl, rows in ((4, 8192), (5, 4096), (6, 4096), (7, 4096), (8, 4096)):
    env = dict(os.environ, PFLU_MC_MAXCL=str(maxcl), PFLU_MC_ROWS=str(rows))
    try:
        out = subprocess.run([sys.executable, "tools/panel_sweep.py", "--m", "32768,16384", "--kernel", "4", "--reps", "5"],
                             env=env, capture_output=True, text=True, timeout=60).stdout
    except subprocess.TimeoutExpired:
        out = "TIMEOUT\n"
    print(f"== maxcl {maxcl} rows/cluster {rows}\n{out}", flush=True)
