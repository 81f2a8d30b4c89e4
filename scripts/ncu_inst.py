"""Instructions executed and stall samples per CUDA source line of one kernel.

    python scripts/ncu_inst.py report.ncu-rep kernel_regex [n]
"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kre}", "-c", "1"], capture_output=True, text=True).stdout
rows = [r for r in csv.reader(io.StringIO(out)) if len(r) > 8 and r[0].isdigit()]
num = lambda x: int(x) if x.isdigit() else 0
tot_i = sum(num(r[7]) for r in rows)
tot_s = sum(num(r[4]) for r in rows)
print(f"warp instructions {tot_i}, stall samples {tot_s}")
for r in sorted(rows, key=lambda r: -num(r[7]))[:n]:
    print(f"{100 * num(r[7]) / max(tot_i, 1):5.1f}% inst {100 * num(r[4]) / max(tot_s, 1):5.1f}% stall  L{r[0]:>4} {r[1].strip()[:100]}")
