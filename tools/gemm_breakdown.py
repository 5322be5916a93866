import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i,r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
K, G, V, U = h.index("Kernel Name"), h.index("Grid Size"), h.index("Metric Value"), h.index("Metric Unit")
d = collections.defaultdict(list)
for r in rows[hi+1:]:
    if "gemm_tc" in r[K]:
        v = float(r[V].replace(",",""))
        v = v/1e3 if r[U].startswith("n") else v
        name = r[K].split("<")[1].split(">")[0] if "<" in r[K] else "?"
        d[(name, r[G])].append(v)
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(k, len(v), f"avg {sum(v)/len(v):.1f} us  total {sum(v)/1e3:.1f} ms  min {min(v):.1f} max {max(v):.1f}")
