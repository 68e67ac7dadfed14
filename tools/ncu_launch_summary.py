"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

  python tools/ncu_launch_summary.py gpurun_out/launches.csv [top]
Per-launch ncu times are cold-cache and serialised: compare SHARES of the step, not absolutes.
Launches are grouped by kernel AND grid size, so one template instantiation used on two
hierarchy levels (e.g. the level-0 and level-1 smoother) shows as two lines, as in bench.py's
per-kernel CUDA-event profile.
"""
import collections
import csv
import re
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = [l for l in open(path) if l.startswith('"')]
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in csv.DictReader(rows):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    name = re.sub(r"\(.*$", "", name)  # drop the parameter list, keep template args
    name = f"{name}  grid {r.get('Grid Size', '?').split(',')[0].strip('( ')}"
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"{sum(cnt.values())} launches, {T:.2f} ms total (ncu, serialised)")
print(f"{'share':>6s} {'ms':>9s} {'launches':>8s}  kernel")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:top]:
    try:
        print(f"{v / T:6.3f} {v:9.3f} {cnt[k]:8d}  {k[:170]}")
    except BrokenPipeError:
        break
