"""Top source lines of one kernel by warp instructions executed (ncu source page).

    python scripts/ncu_hotlines.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kre}", "-c", "1"], capture_output=True, text=True).stdout
cur, rows, tot, hdr = None, [], 0, None
for r in csv.reader(io.StringIO(out)):
    if r and r[0] in ("File Name", "File Path"):
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        d = dict(zip(hdr, r))
        n = d.get("Instructions Executed", "0")
        n = int(float(n)) if n.replace(".", "").isdigit() else 0
        smp = d.get("Warp Stall Sampling (All Samples)", "0")
        smp = int(float(smp)) if smp.replace(".", "").isdigit() else 0
        tot += n
        rows.append((n, smp, cur, int(r[0]), r[1].strip()[:100]))
tsmp = sum(x[1] for x in rows)
print(f"warp instructions {tot}, stall samples {tsmp}   (inst %, sample %)")
for n, smp, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100 * n / max(tot, 1):5.1f}% {100 * smp / max(tsmp, 1):5.1f}% {f}:{ln:<5d} {src}")
