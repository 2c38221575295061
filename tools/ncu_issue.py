"""Issue-side roofline of every hot-path kernel in an ncu --set full report:
thread-instructions per element, issue-slot utilisation, IPC and DRAM bytes
per launch -- merged into profiles/issue.json under "config<N>" (bench.py
reports it next to each op's HBM roofline fraction: for this block format
the instruction issue, not HBM, is the ceiling).

    python tools/ncu_issue.py <report.ncu-rep> <config> <elements> [note]
"""
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_traffic import op_of  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "issue.json")

WANT = {
    "smsp__inst_executed.sum": "warp_inst",
    "sm__inst_executed.avg.per_cycle_active": "ipc",
    "sm__instruction_throughput.avg.pct_of_peak_sustained_active": "issue_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_slots_busy_pct",
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9,
         "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9}


def main():
    rep, config, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    note = sys.argv[4] if len(sys.argv) > 4 else os.path.basename(rep)
    text = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(WANT)],
                          capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(text)))
    h, units = r[0], r[1]
    ki = h.index("Kernel Name")
    res = {}
    for row in r[2:]:
        op = op_of(row[ki])
        if not op:
            continue
        m = {}
        for metric, key in WANT.items():
            if metric not in h:
                continue
            i = h.index(metric)
            try:
                v = float(row[i].replace(",", ""))
            except ValueError:
                continue
            m[key] = v * SCALE.get(units[i], 1.0)
        e = {"thread_inst_per_element": round(m.get("warp_inst", 0) * 32 / n, 2),
             "issue_slots_busy_pct": round(m.get("issue_slots_busy_pct", 0), 1),
             "ipc": round(m.get("ipc", 0), 2),
             "duration_us": round(m.get("duration", 0) * 1e6, 1),
             "dram_bytes": int(m.get("dram_read", 0) + m.get("dram_write", 0))}
        res[op] = e                     # the last launch of each kernel
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    data[f"config{config}"] = res
    data.setdefault("sources", {})[f"config{config}"] = note
    json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
