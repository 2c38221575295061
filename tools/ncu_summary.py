"""Summarise an ncu --csv launch list: last launch of each kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    agg.setdefault((r[idi], r[ki]), {})[r[mi]] = r[vi]
last = collections.OrderedDict()
for (i, name), m in agg.items():
    last.setdefault(name, []).append(m)
only = sys.argv[2] if len(sys.argv) > 2 else ""
for name, ms in last.items():
    if only and only not in name:
        continue
    m = ms[-1]
    short = name.split("(")[0][-60:]
    t = float(m.get("gpu__time_duration.sum", "nan").replace(",", ""))
    rd = float(m.get("dram__bytes_read.sum", "0").replace(",", ""))
    wr = float(m.get("dram__bytes_write.sum", "0").replace(",", ""))
    inst = m.get("smsp__inst_executed.sum", "")
    print(f"{short:60s} n={len(ms):2d} t={t/1000:8.1f}us dram_rd={rd/1e6:8.2f}MB wr={wr/1e6:7.2f}MB inst={inst}")
