"""Per-kernel totals of an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import collections
import csv
import sys

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"'))
        if r["Metric Name"] == "gpu__time_duration.sum"]
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows:
    name = r["Kernel Name"].replace("(anonymous namespace)::", "").split("(")[0]
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    v *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(unit, 1e-6)
    tot[name] += v
    cnt[name] += 1
allms = sum(tot.values())
peak = sum(v for k, v in tot.items() if "k_dfma" in k)
print(f"launches={len(rows)} total_ms={allms:.3f}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    excl = 0.0 if "k_dfma" in k else v / max(allms - peak, 1e-9)
    print(f"{k[:60]:60s} launches={cnt[k]:4d} total_ms={v:9.3f} share={100 * v / allms:5.1f}% "
          f"share_excl_peak_bench={100 * excl:5.1f}%")
