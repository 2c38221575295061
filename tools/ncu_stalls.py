"""Stall reasons of one kernel in an ncu --set full report, split by source
line ranges (e.g. the roles of a warp-specialised kernel).

    python tools/ncu_stalls.py rep.ncu-rep <launch index> name=file:lo-hi[,file:lo-hi] ...
Lines not matched by any range go to "other"."""
import collections
import csv
import io
import subprocess
import sys

rep, idx = sys.argv[1], int(sys.argv[2])
groups = []
for spec in sys.argv[3:]:
    name, ranges = spec.split("=", 1)
    rr = []
    for r in ranges.split(","):
        f, span = r.split(":")
        lo, hi = span.split("-")
        rr.append((f, int(lo), int(hi)))
    groups.append((name, rr))
text = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                       "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(text)))
fname, hdr = None, None
acc = collections.defaultdict(lambda: collections.Counter())
inst = collections.Counter()
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or r[2] != "-":
        continue
    try:
        line = int(r[0])
    except ValueError:
        continue
    g = "other"
    for name, rr in groups:
        if any(fname == f and lo <= line <= hi for f, lo, hi in rr):
            g = name
            break
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                acc[g][h[6:]] += int(r[i])
            except ValueError:
                pass
    try:
        inst[g] += int(r[hdr.index("Instructions Executed")])
    except ValueError:
        pass
tot_all = sum(sum(c.values()) for c in acc.values()) or 1
ti = sum(inst.values()) or 1
for g, c in sorted(acc.items(), key=lambda x: -sum(x[1].values())):
    t = sum(c.values()) or 1
    top = ", ".join(f"{k} {100 * v / t:.0f}%" for k, v in c.most_common(7))
    print(f"{g:10s} samples {100 * t / tot_all:5.1f}%  inst {100 * inst[g] / ti:5.1f}%  | {top}")
