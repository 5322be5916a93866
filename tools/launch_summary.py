"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel name."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tot = collections.defaultdict(float); cnt = collections.Counter()
seen = 0
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    seen += 1
    if seen <= skip:
        continue
    name = r[ki].split("(")[0].split("<")[0][:60]
    v = float(r[vi].replace(",", ""))
    unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "nsecond"
    v = v / 1e3 if unit.startswith("n") else (v if unit.startswith("u") else v * 1e3)
    tot[name] += v; cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':60s} {'n':>6s} {'total_ms':>10s} {'avg_us':>9s} {'share':>6s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:60s} {cnt[k]:6d} {v/1e3:10.2f} {v/cnt[k]:9.1f} {100*v/T:5.1f}%")
print(f"{'TOTAL':60s} {sum(cnt.values()):6d} {T/1e3:10.2f}")
