#!/usr/bin/env python
"""Print the key ncu metrics of every kernel in a report (one line per metric)."""
import csv
import io
import subprocess
import sys

WANT = ("Duration", "Elapsed Cycles", "Registers Per Thread", "Dynamic Shared Memory Per Block", "Achieved Occupancy",
        "Theoretical Occupancy", "Block Limit Shared Mem", "Block Limit Registers", "Issue Slots Busy",
        "Executed Ipc Active", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler",
        "Active Warps Per Scheduler", "Local Memory Spilling Requests", "Avg. Active Threads Per Warp")
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
seen = set()
for d in csv.DictReader(io.StringIO(out)):
    m = d.get("Metric Name", "")
    key = (d.get("Kernel Name"), d.get("ID"), m)
    if m in WANT and key not in seen:
        seen.add(key)
        print(f'{d.get("Kernel Name","")[:28]:28s} {d.get("ID",""):>3s} {m:40s} {d.get("Metric Value","")} {d.get("Metric Unit","")}')
