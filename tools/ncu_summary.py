"""Summarise an .ncu-rep (details page) into a compact text table: python tools/ncu_summary.py rep [metric filter]."""
import csv
import subprocess
import sys

WANT = ['Duration', 'Registers Per Thread', 'Achieved Occupancy', 'Theoretical Occupancy', 'Compute (SM) Throughput',
        'Memory Throughput', 'DRAM Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate', 'Executed Ipc Active',
        'Issue Slots Busy', 'Avg. Active Threads Per Warp', 'Avg. Not Predicated Off Threads Per Warp',
        'Warp Cycles Per Issued Instruction', 'No Eligible', 'Grid Size', 'Block Size', 'Dynamic Shared Memory Per Block',
        'Block Limit Registers', 'Block Limit Shared Mem', 'Waves Per SM', 'SM Frequency', 'DRAM Frequency']
out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'details', '--csv'], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
ki, mi, vi, ui, idi = (h.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
extra = sys.argv[2:] if len(sys.argv) > 2 else []
for x in r[1:]:
    if x[mi] in WANT or any(e in x[mi] for e in extra):
        print(x[idi], x[ki][:28], '|', x[mi], '=', x[vi], x[ui])
