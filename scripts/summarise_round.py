"""Copy the judged measurement summaries of one scripts/measure_round.sh run into profiles/.

    python scripts/summarise_round.py r01
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"


def last_json_line(path):
    with open(path) as f:
        lines = [ln for ln in f.read().splitlines() if ln.strip().startswith("{")]
    return json.loads(lines[-1])


def run(cmd):
    return subprocess.run(cmd, capture_output=True, text=True).stdout


b = last_json_line(os.path.join(G, "bench.json"))
json.dump(b, open(os.path.join(P, f"{tag}_bench.json"), "w"), indent=1)
r = last_json_line(os.path.join(G, "bench_ref.json"))
json.dump(r, open(os.path.join(P, f"{tag}_bench_reference.json"), "w"), indent=1)
open(os.path.join(P, f"{tag}_bench_launches.txt"), "w").write(
    run([sys.executable, os.path.join(ROOT, "scripts", "launch_table.py"), os.path.join(G, "bench_launches.csv")]))
for v in (0, 1, 2):
    src = os.path.join(G, f"frame_v{v}.txt")
    if os.path.exists(src):
        shutil.copy(src, os.path.join(P, f"{tag}_frame_view{v}_launches.txt"))
summ = ""
for rep in ("ncu_blend", "ncu_top", "ncu_sort", "ncu_up"):
    path = os.path.join(G, rep + ".ncu-rep")
    if os.path.exists(path):
        summ += run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), path])
open(os.path.join(P, f"{tag}_ncu_summary.txt"), "w").write(summ)
# DRAM bytes per k_blend launch (near / mid / far), the roofline's `traffic`
raw = run(["ncu", "-i", os.path.join(G, "ncu_blend.ncu-rep"), "--page", "raw", "--csv"])
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
per = []
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = float(d["dram__bytes_read.sum"]) * scale[units[hdr.index("dram__bytes_read.sum")]]
    wr = float(d["dram__bytes_write.sum"]) * scale[units[hdr.index("dram__bytes_write.sum")]]
    per.append(rd + wr)
if len(per) == 3:
    json.dump({"kernel": "k_blend", "per_launch_bytes": sum(per) / 3,
               "per_view_bytes": dict(zip(("near", "mid", "far"), per)),
               "source": f"ncu --set full --clock-control none, config 3 near/mid/far, one launch each "
                         f"(profiles/{tag}_ncu_summary.txt)"},
              open(os.path.join(P, "blend_dram_bytes.json"), "w"), indent=1)
print(json.dumps({k: b.get(k) for k in ("value", "ms_per_step", "stage_ms", "e2e", "gpu_launches")}, indent=1))
