"""Per-launch table (duration, DRAM bytes) of one profiled frame.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --nvtx \
        --nvtx-include "frame/" --clock-control none --csv --log-file F.csv python scripts/profile_frame.py cfg3 2
    python scripts/frame_kernels.py F.csv
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, per = None, {}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        k = per.setdefault(d["ID"], {"name": d["Kernel Name"].split("(")[0][:34], "grid": d["Grid Size"]})
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}.get(unit, 1)
        k[d["Metric Name"]] = v * scale
tot = 0.0
print(f"{'id':>4} {'kernel':34s} {'grid':>14s} {'us':>9s} {'rd MB':>9s} {'wr MB':>9s} {'GB/s':>7s}")
for i, k in sorted(per.items(), key=lambda x: int(x[0])):
    t = k.get("gpu__time_duration.sum", 0.0)
    rd, wr = k.get("dram__bytes_read.sum", 0.0), k.get("dram__bytes_write.sum", 0.0)
    tot += t
    print(f"{i:>4} {k['name']:34s} {k['grid']:>14s} {t / 1e3:9.1f} {rd / 1e6:9.1f} {wr / 1e6:9.1f} "
          f"{(rd + wr) / max(t, 1):7.0f}")
print(f"total {tot / 1e6:.3f} ms (serialised)")
