import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i,r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]; data = rows[hdr+1:]
ki = h.index("Kernel Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
tot = collections.defaultdict(float); cnt = collections.Counter()
scale = {"nsecond":1e-3, "usecond":1.0, "msecond":1e3, "ns":1e-3, "us":1.0, "ms":1e3}
for r in data:
    v = float(r[vi].replace(",","")) * scale.get(r[ui], 1.0)
    name = r[ki].split("(")[0]
    name = name.replace("void ", "").replace("fhe::", "").replace("<unnamed>::", "")
    tot[name] += v; cnt[name] += 1
T = sum(tot.values())
for k,v in sorted(tot.items(), key=lambda x:-x[1]):
    print(f"{k[:60]:60s} {cnt[k]:5d} {v:10.1f} us {100*v/T:5.1f}%  avg {v/cnt[k]:8.2f}")
print(f"total {T:.1f} us over {sum(cnt.values())} launches")
