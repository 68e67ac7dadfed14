"""Copy one evidence run (tools/_bench_evidence.sh <tag>, merged into gpurun_out/) into
profiles/: the bench JSON line, the ncu launch list (gz + summary grouped by kernel and
grid) and the three ncu --set full captures, and rebuild profiles/traffic.json (the DRAM
bytes per launch bench.py reports as roofline.traffic / spmv.traffic).

  python tools/refresh_evidence.py r01f
"""
import csv
import gzip
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
line = [l for l in open(os.path.join(G, f"{tag}_bench.log")) if l.startswith("{")][-1]
open(os.path.join(P, "r01_bench_cfg5.json"), "w").write(line)
with open(os.path.join(G, f"{tag}_launches.csv"), "rb") as f, gzip.open(os.path.join(P, "r01_ncu_launches_cfg5.csv.gz"), "wb") as g:
    shutil.copyfileobj(f, g)
summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_launch_summary.py"),
                       os.path.join(G, f"{tag}_launches.csv"), "40"], capture_output=True, text=True).stdout
open(os.path.join(P, "r01_ncu_launches_cfg5_summary.txt"), "w").write(summ)
SC = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
TU = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9}
caps = [("spmv_b4_f64xf32@cfg5", "top", "r01_ncu_full_cfg5_outer_spmv_details.csv", "outer 4x4 fp64 x fp32 SpMV, one launch"),
        ("smooth_b3_f32xf32@cfg5", "smooth", "r01_ncu_full_cfg5_l0_smooth_details.csv", "level-0 3x3 fp32 smoother, first launch"),
        ("spmv_cfg2_b4_f32xf64", "spmv", "r01_ncu_full_cfg2_spmv_details.csv", "cfg-2 4x4 fp32 x fp64 SpMV, one launch")]
traffic = {}
for key, f, dst, what in caps:
    shutil.copy(os.path.join(G, f"{tag}_ncu_{f}_details.csv"), os.path.join(P, dst))
    r = list(csv.reader(open(os.path.join(G, f"{tag}_ncu_{f}_raw.csv"))))
    h, units, d = r[0], r[1], dict(zip(r[0], r[2]))
    rd = float(d["dram__bytes_read.sum"]) * SC[units[h.index("dram__bytes_read.sum")]]
    wr = float(d["dram__bytes_write.sum"]) * SC[units[h.index("dram__bytes_write.sum")]]
    traffic[key] = {"kernel": d["Kernel Name"], "dram_bytes_read": rd, "dram_bytes_write": wr, "traffic": rd + wr,
                    "ncu_duration_s": float(d["gpu__time_duration.sum"]) * TU[units[h.index("gpu__time_duration.sum")]],
                    "source": f"profiles/{dst}",
                    "capture": f"ncu --set full --clock-control none: {what} (tools/_bench_evidence.sh {tag})"}
json.dump(traffic, open(os.path.join(P, "traffic.json"), "w"), indent=1)
print(line.strip()[:200])
print(summ.splitlines()[0])
