"""DRAM traffic per launch of each hot-path kernel from an ncu report (or an
ncu --csv launch list with dram__bytes_read.sum / dram__bytes_write.sum),
merged into profiles/traffic.json under "config<N>" -- the `traffic` field
of bench.py's roofline object.

    python tools/ncu_traffic.py <report.ncu-rep | launches.csv> <config> [source note]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "traffic.json")

KERNEL_OP = [
    ("compress_f32_kernel", "compress"),
    ("recode_kernel<0>", "scalar_mul"),
    ("recode_kernel<(int)0>", "scalar_mul"),
    ("decode_pipe_kernel<0>", "mean"),
    ("decode_pipe_kernel<(int)0>", "mean"),
    ("decode_pipe_kernel<1>", "variance"),
    ("decode_pipe_kernel<(int)1>", "variance"),
    ("decode_pipe_kernel<2>", "decompress"),
    ("decode_pipe_kernel<(int)2>", "decompress"),
    ("negate32_kernel", "negate"),
    ("sadd_kernel", "scalar_add"),
    ("minmax_f32_kernel", "minmax"),
]


def op_of(name):
    for k, op in KERNEL_OP:
        if k in name:
            return op
    return None


def _num(v):
    return float(str(v).replace(",", ""))


def rows(path):
    if path.endswith(".ncu-rep"):
        text = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics",
                               "dram__bytes_read.sum,dram__bytes_write.sum"],
                              capture_output=True, text=True).stdout
        r = list(csv.reader(io.StringIO(text)))
        h = r[0]
        units = r[1]
        ki = h.index("Kernel Name")
        rd, wr = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        for x in r[2:]:
            yield x[ki], _num(x[rd]) * scale.get(units[rd], 1) + _num(x[wr]) * scale.get(units[wr], 1)
        return
    # ncu --csv launch list: one row per (launch, metric)
    r = list(csv.reader(open(path)))
    h = next(x for x in r if "Metric Name" in x)
    start = r.index(h) + 1
    ki, mi, vi, ui = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    ii = h.index("ID")
    acc = {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for x in r[start:]:
        if len(x) <= vi or x[mi] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            continue
        key = (x[ii], x[ki])
        acc[key] = acc.get(key, 0.0) + _num(x[vi]) * scale.get(x[ui], 1)
    for (_, name), v in acc.items():
        yield name, v


def main():
    path, config = sys.argv[1], int(sys.argv[2])
    note = sys.argv[3] if len(sys.argv) > 3 else os.path.basename(path)
    last = {}
    for name, b in rows(path):
        op = op_of(name)
        if op:
            last[op] = int(b)           # the last launch of each kernel
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    data[f"config{config}"] = last
    data.setdefault("sources", {})[f"config{config}"] = note
    json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)
    print(json.dumps(last, indent=1))


if __name__ == "__main__":
    main()
