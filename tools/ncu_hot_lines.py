"""Aggregate ncu source-page metrics per CUDA source line (needs -lineinfo + --import-source)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res = []
fname = "?"
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "Function Name") and len(r) >= 8:
        try:
            samples = float(r[4] or 0)
            inst = float(r[7] or 0)
        except ValueError:
            continue
        res.append((samples, inst, f"{fname}:{r[0]}", r[1].strip()[:100]))
ts = sum(x[0] for x in res) or 1
ti = sum(x[1] for x in res) or 1
for s, i, loc, src in sorted(res, reverse=True)[:top]:
    print(f"{100 * s / ts:5.1f}% samples {100 * i / ti:5.1f}% inst {loc:28s} {src}")
