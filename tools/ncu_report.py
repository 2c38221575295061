"""Summarise one kernel of an ncu --set full report: key metrics, stall
reasons, per-source-line instruction counts and stall samples.

    python tools/ncu_report.py rep.ncu-rep [launch_index] [top_lines]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


det = list(csv.reader(io.StringIO(ncu("--page", "details", "--csv"))))
h = det[0]
ki, mi, vi, ui, ii = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
ids = sorted({r[ii] for r in det[1:]}, key=int)
want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "No Eligible", "Eligible Warps Per Scheduler", "Active Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "L2 Hit Rate",
        "Dynamic Shared Memory Per Block", "Grid Size", "Local Memory Spilling Requests"]
sel = ids[idx]
for r in det[1:]:
    if r[ii] == sel and r[mi] in want:
        print(f"  {r[mi]:38s} {r[vi]} {r[ui]}")
        name = r[ki]
print("kernel:", name[:100])
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hr = raw[0]
row = [r for r in raw[2:]][idx]
st = {}
for i, nm in enumerate(hr):
    if nm.startswith("smsp__average_warp_latency_issue_stalled_") and nm.endswith(".ratio"):
        try:
            st[nm.replace("smsp__average_warp_latency_issue_stalled_", "").replace(".ratio", "")] = float(row[i].replace(",", ""))
        except ValueError:
            pass
    if "dram__bytes_read.sum" == nm or "dram__bytes_write.sum" == nm:
        print(f"  {nm} {row[i]}")
tot = sum(st.values()) or 1
print("stall reasons (share of warp cycles):", ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]))
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "cuda,sass",
                                      "--launch-skip", str(idx), "--launch-count", "1"))))
hdr = None
fname = None
lines = []
for r in src:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    try:
        n = int(r[hdr.index("Instructions Executed")])
        s = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except (ValueError, IndexError):
        continue
    if n or s:
        lines.append((n, s, f"{fname}:{r[0]}", r[1].strip()[:80]))
ti = sum(l[0] for l in lines) or 1
ts = sum(l[1] for l in lines) or 1
print(f"-- top lines by stall samples (total inst {ti/1e6:.1f}M)")
for n, s, loc, code in sorted(lines, key=lambda l: -l[1])[:top]:
    print(f"  {100*s/ts:5.1f}% st {100*n/ti:5.1f}% in  {loc:26s} {code}")
