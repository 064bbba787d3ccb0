"""Hot source lines of a kernel from an `ncu --set full --import-source on` report: warp-stall samples
aggregated per CUDA source line (mixed cuda,sass page), top N printed with the line text.

    python tools/ncu_source_hot.py report.ncu-rep [N]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
samples = collections.Counter()
texts = {}
fname = None
total = 0
hdr = None
cur = None
for row in csv.reader(io.StringIO(raw)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) < 5:
        continue
    # rows: a source line (Line No, Source, then empty sass cols) or sass rows under it
    if row[0] and row[0].isdigit():
        cur = (fname, int(row[0]))
        texts[cur] = row[1].strip()
        try:
            v = int(row[4] or 0)
        except ValueError:
            v = 0
        samples[cur] += v
        total += v
print(f"total stall samples {total}")
for (f, ln), v in samples.most_common(top):
    print(f"{v:8d} {100.0 * v / max(1, total):5.1f}%  {f}:{ln}  {texts[(f, ln)][:110]}")
