"""Brief of an ncu --page details/raw export: SOL, occupancy, stall reasons per kernel."""
import csv, sys
tag = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/{tag}_details.csv")))
h = rows[0]
ki, si, ni, ui, vi = (h.index(x) for x in ("Kernel Name", "Section Name", "Metric Name", "Metric Unit", "Metric Value"))
keep = {"Duration", "DRAM Throughput", "Memory Throughput", "SM Active Cycles", "Elapsed Cycles", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Issued Warp Per Scheduler", "Eligible Warps Per Scheduler", "Active Warps Per Scheduler",
        "Registers Per Thread", "Grid Size", "Block Size", "Compute (SM) Throughput", "Mem Pipes Busy"}
for r in rows[1:]:
    if r[ni] in keep:
        print(r[ki][:24], "|", r[ni], r[vi], r[ui])
raw = list(csv.reader(open(f"gpurun_out/{tag}_raw.csv")))
hh = raw[0]
for r in raw[2:]:
    print(r[hh.index("Kernel Name")][:40], "instr", r[hh.index("smsp__inst_executed.sum")] if "smsp__inst_executed.sum" in hh else "")
    vals = [(x, r[hh.index(x)]) for x in hh if "smsp__pcsamp_warps_issue_stalled" in x and not x.endswith("not_issued")]
    vals = [(x, float(v)) for x, v in vals if v.replace(".", "", 1).isdigit()]
    tot = sum(v for _, v in vals) or 1
    print("  stalls:", ", ".join(f"{x.split('stalled_')[1]} {v / tot:.0%}" for x, v in sorted(vals, key=lambda z: -z[1])[:7]))
