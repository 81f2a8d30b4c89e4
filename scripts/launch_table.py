"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per-kernel total time and share."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, out = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            out.append((d["Kernel Name"].split("(")[0], float(d["Metric Value"].replace(",", "")), d["Grid Size"]))
tot = sum(v for _, v, _ in out)
agg = {}
for n, v, g in out:
    a = agg.setdefault(n, [0.0, 0, g]); a[0] += v; a[1] += 1
print(f"{'kernel':28s} {'us':>10s} {'share':>6s} {'launches':>8s}")
for n, (v, c, g) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{n:28s} {v/1e3:10.1f} {100*v/tot:5.1f}% {c:8d}")
print(f"{'TOTAL':28s} {tot/1e3:10.1f}   ({len(out)} launches, serialised, cold caches)")
