"""Per-kernel totals of an ncu launch list (gpu__time_duration.sum, --csv) and the launch
sequence of its last evaluation (everything after the second-to-last k_quad).
    python tools/launch_seq.py gpurun_out/launches.csv [--seq]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
for k, r in enumerate(rows):
    if "Kernel Name" in r:
        h, start = r, k
        break
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
seq = []
for r in rows[start + 1:]:
    if len(r) <= vi:
        continue
    nm = r[ki].replace("(anonymous namespace)::", "").replace("void ", "")
    m = re.search(r"(k_[a-z0-9_]+|scvt_[a-z0-9_]+|cub::\w+|at::\w+|\w+)\s*[<(]", nm)
    name = m.group(1) if m else nm[:40]
    v = float(r[vi].replace(",", ""))
    if r[ui] == "ns":
        v /= 1e3
    agg[name][0] += 1
    agg[name][1] += v
    seq.append((name, v))
tot = sum(v[1] for v in agg.values())
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{n[:46]:46s} {c:5d} {t:10.1f} us {t / c:9.1f} us/launch {100 * t / tot:5.1f}%")
if "--seq" in sys.argv:
    idx = [k for k, (n, v) in enumerate(seq) if n == "k_quad"]
    a, b = idx[-2], idx[-1]
    for n, v in seq[a + 1:b + 1]:
        print(f"   {n:30s} {v:9.1f}")
