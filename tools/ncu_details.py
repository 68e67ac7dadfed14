"""Key metrics of an ncu --page details --csv export (one or more kernels).

  python tools/ncu_details.py file.csv [extra metric names ...]
"""
import csv
import sys

WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Registers Per Thread', 'No Eligible', 'Grid Size', 'Eligible Warps Per Scheduler',
        'Active Warps Per Scheduler', 'Issued Warp Per Scheduler', 'L2 Cache Throughput', 'L1/TEX Cache Throughput',
        'Mem Busy', 'Max Bandwidth', 'Block Limit Registers'] + sys.argv[2:]
rows = [r for r in csv.reader(open(sys.argv[1]))]
h = rows[0]
ki, mi, vi, ui = (h.index(k) for k in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit'))
last = None
for r in rows[1:]:
    if r[ki] != last:
        last = r[ki]
        print(last[:110])
    if r[mi] in WANT:
        print(f'   {r[mi]:32s} {r[vi]} {r[ui]}')
