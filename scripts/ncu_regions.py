"""Instructions executed per source file / line range of one kernel (ncu source page).

    python scripts/ncu_regions.py report.ncu-rep kernel_regex file.cu name:lo-hi ...
"""
import csv
import io
import subprocess
import sys

rep, kre, fname = sys.argv[1], sys.argv[2], sys.argv[3]
ranges = []
for a in sys.argv[4:]:
    name, lohi = a.split(":")
    lo, hi = lohi.split("-")
    ranges.append((name, int(lo), int(hi)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kre}", "-c", "1"], capture_output=True, text=True).stdout
cur, agg, tot = None, {}, 0
num = lambda x: int(x) if x.isdigit() else 0   # noqa: E731
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0].isdigit():
        ln, n = int(r[0]), num(r[7])
        tot += n
        reg = cur
        if cur == fname:
            reg = next((nm for nm, lo, hi in ranges if lo <= ln <= hi), f"{fname}:other")
        agg[reg] = agg.get(reg, 0) + n
print(f"warp instructions {tot}")
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"  {k:24s} {100 * v / max(tot, 1):5.1f}%")
