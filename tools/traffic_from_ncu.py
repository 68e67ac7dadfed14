"""Write profiles/traffic.json (read by bench.py as roofline.traffic) from ncu --set full raw CSV
captures: DRAM bytes read + written per launch of each captured kernel.

  python tools/traffic_from_ncu.py TAG      (reads gpurun_out/TAG_ncu_{top,smooth,...}_raw.csv)
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG = sys.argv[1]
# bench key -> (capture name, description)
KEYS = {
    "spmv_b4_f64xf32@cfg5": ("top", "outer 4x4 fp64 x fp32 SpMV, one launch"),
    "smooth_b3_f32xf32@cfg5": ("smooth", "level-0 3x3 fp32 smoother, first launch"),
    "residual_b3_f32xf32@cfg5": ("resid", "level-0 3x3 fp32 residual, first launch"),
    "spmv_b3_f32xf32@cfg5": ("p0", "level-0 prolongation P0 (operand ahead of the row), one launch"),
    "spmv_M_b3_f32xf32@cfg5": ("r0m", "restriction R0 + the level-1 pre-smoothing x = M f (fused K4a)"),
    "split_M_b4_f64xf32@cfg5": ("splitm", "K9 split + the level-0 pre-smoothing (fused K4a)"),
    "schur_u_M_b3_f32xf32@cfg5": ("schurum", "K11 B^T update + the level-0 pre-smoothing (fused K4a)"),
    "schur_p_b3_f32xf32@cfg5": ("schurp", "K10 Schur B product"),
    "smooth_join_b3_f32xf32@cfg5": ("smoothjoin", "level-0 last post-smoothing + join z = (u, p) (fused K9')"),
    "mdot_b25_f16@cfg5": ("mdot16", "GMRES pass-1 multi-dot on the fp16 shadow (R28), k >= 25"),
    "cgs_update_dots_nrm_b25_f64@cfg5": ("update", "GMRES pass-2 update + dots + norm, k >= 25"),
    "spmv_cfg2_b4_f32xf64": ("spmv", "cfg-2 4x4 fp32 x fp64 SpMV, one launch"),
}


def unit_scale(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[u]


out = {}
for key, (cap, what) in KEYS.items():
    path = os.path.join(ROOT, "gpurun_out", f"{TAG}_ncu_{cap}_raw.csv")
    if not os.path.exists(path):
        continue
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}

    def get(m):
        v, u = d[m]
        return float(v.replace(",", "")) * unit_scale(u)

    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    v, u = d["gpu__time_duration.sum"]
    dur = float(v.replace(",", "")) * {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}[u]
    out[key] = {"kernel": d["Kernel Name"][0], "dram_bytes_read": rd, "dram_bytes_write": wr, "traffic": rd + wr,
                "ncu_duration_s": dur, "source": f"profiles/{TAG}_ncu_{cap}_details.csv",
                "capture": f"ncu --set full --clock-control none: {what} (tools/_evidence_r02.sh {TAG})"}
json.dump(out, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
for k, v in out.items():
    print(f"{k:28s} {v['traffic'] / 1e9:8.3f} GB  {v['ncu_duration_s'] * 1e3:7.3f} ms  {v['traffic'] / v['ncu_duration_s'] / 1e12:5.2f} TB/s")
