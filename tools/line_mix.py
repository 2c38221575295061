"""Per-CUDA-line instruction counts / stall samples from
`ncu --page source --csv --print-source cuda,sass` output."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
topn = int(sys.argv[3]) if len(sys.argv) > 3 else 40
fname = None
out = []
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[2] != "-":          # SASS rows carry an address; CUDA rows have '-'
        continue
    try:
        inst = int(r[hdr.index("Instructions Executed")])
        smp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except (ValueError, IndexError):
        continue
    if inst or smp:
        out.append((inst, smp, f"{fname}:{r[0]}", r[1].strip()[:90]))
tot_i = sum(o[0] for o in out)
tot_s = sum(o[1] for o in out)
print(f"total inst/unit {tot_i / norm:.1f}  samples {tot_s}")
for inst, smp, loc, src in sorted(out, key=lambda o: -o[0])[:topn]:
    print(f"{inst / norm:7.2f} {100 * smp / max(tot_s, 1):5.1f}%  {loc:22s} {src}")
