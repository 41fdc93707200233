"""Per-launch table of an ncu --csv launch list (--metrics gpu__time_duration.sum[,dram...]).

    python tools/launch_table.py gpurun_out/x/launches.csv [last_n]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, mi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name"), h.index("ID")
gi = h.index("Grid Size") if "Grid Size" in h else None
t = collections.OrderedDict()
for r in rows[hdr + 1:]:
    e = t.setdefault(r[ii], {"k": r[ki].split("(")[0][:40], "grid": r[gi] if gi is not None else ""})
    try:
        e[r[mi]] = float(r[vi].replace(",", ""))
    except ValueError:
        pass
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for k, v in list(t.items())[-n:]:
    print("%4s %-40s %-14s %9.1f us  rd %8.1f MB  wr %8.1f MB" % (
        k, v["k"], v["grid"], v.get("gpu__time_duration.sum", 0) / 1e3, v.get("dram__bytes_read.sum", 0) / 1e6,
        v.get("dram__bytes_write.sum", 0) / 1e6))
