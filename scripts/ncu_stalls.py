"""Top source lines of one kernel by warp-stall samples, with their two leading stall reasons.

    python scripts/ncu_stalls.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kre}", "-c", "1"], capture_output=True, text=True).stdout
hdr, rows, cur = None, [], None
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        rows.append((cur, r))
if not hdr:
    sys.exit("no source page")
idx = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
num = lambda v: int(v) if v.isdigit() else 0   # noqa: E731
tot = {s: sum(num(r[idx[s]]) for _, r in rows) for s in stalls}
T = max(1, sum(tot.values()))
print("stall mix:", ", ".join(f"{k[6:]} {100 * v / T:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
res = []
for f, r in rows:
    smp = sum(num(r[idx[s]]) for s in stalls)
    lead = sorted(((num(r[idx[s]]), s[6:]) for s in stalls), reverse=True)[:2]
    res.append((smp, f, int(r[0]), r[1].strip()[:80], lead))
for smp, f, ln, src, lead in sorted(res, reverse=True)[:top]:
    print(f"{100 * smp / T:5.1f}% {f}:{ln:<5d} {src}  [{', '.join(f'{n} {100 * c / max(smp, 1):.0f}%' for c, n in lead)}]")
