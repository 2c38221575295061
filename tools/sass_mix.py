"""Opcode mix + stall samples of one kernel from `ncu --page source --csv --print-source sass`."""
import collections
import csv
import sys

r = list(csv.reader(open(sys.argv[1])))
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
h = r[1]
data = r[2:]
si, ei = h.index("Source"), h.index("Instructions Executed")
smp = h.index("Warp Stall Sampling (All Samples)")
ops, samples = collections.Counter(), collections.Counter()
tot = tots = 0
for x in data:
    try:
        n = int(x[ei])
    except (ValueError, IndexError):
        continue
    toks = x[si].strip().split()
    op = toks[0] if toks else "?"
    if op.startswith("@"):
        op = toks[1]
    base = op.split(".")[0]
    ops[base] += n
    tot += n
    s = int(x[smp] or 0)
    samples[base] += s
    tots += s
print(f"total {tot / norm:.1f} per unit, stall samples {tots}")
for k, v in ops.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 30):
    print(f"{k:10s} {v / norm:7.1f}  samples={samples[k]:6d} ({100 * samples[k] / max(tots, 1):.1f}%)")
