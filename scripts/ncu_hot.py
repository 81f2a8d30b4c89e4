"""Hottest SASS lines of one kernel in an ncu report (stall samples), with the source line.

    python scripts/ncu_hot.py report.ncu-rep kernel_regex [n]
"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda", "-k", f"regex:{kre}",
                      "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if "Address" in r or "# Address" in r or "Source" in r)
hdr = rows[hdr_i]
data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
ia = hdr.index("Warp Stall Sampling (All Samples)")
g = lambda r: int(r[ia]) if r[ia].isdigit() else 0
tot = sum(g(r) for r in data)
print("samples", tot)
cols = [c for c in hdr if c.startswith("stall_") or "Stall" in c]
for i in sorted(sorted(range(len(data)), key=lambda i: -g(data[i]))[:n]):
    r = data[i]
    print(f"{i:5d} {100 * g(r) / max(tot, 1):5.1f}% {r[1][:110]}")
