"""Summarise `ncu --set full` reports (run here, no GPU needed).

    python tools/ncu_summary.py gpurun_out/ncu_*.ncu-rep > profiles/rNN_ncu_summary.md
    python tools/ncu_summary.py --traffic profiles/ncu_traffic.json gpurun_out/ncu_*.ncu-rep

Per launch: duration, DRAM bytes read/written, DRAM throughput, tensor-pipe
activity, SM throughput, achieved occupancy, registers and shared memory.
--traffic also writes {stage: {"dram_bytes_per_launch": ...}} for bench.py's
roofline "traffic" field.
"""
import csv
import io
import json
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"
KEYS = [
    ("time_us", "gpu__time_duration.sum", 1.0),
    ("dram_read_B", "dram__bytes_read.sum", None),
    ("dram_write_B", "dram__bytes_write.sum", None),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("tensor_pct", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("sm_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("occupancy_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    ("regs", "launch__registers_per_thread", 1.0),
    ("smem_dyn_B", "launch__shared_mem_per_block_dynamic", None),
    ("grid", "launch__grid_size", 1.0),
    ("block", "launch__block_size", 1.0),
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1.0, "ns": 1e-3, "ms": 1e3,
        "Kbyte/block": 1e3, "byte/block": 1}
# stage name used by bench.py for each kernel
STAGE = {"k_boxes_crops": "k1_boxes_crops", "k_crops_staged": "k1_boxes_crops", "k_encoder_tc": "k2_encoder",
         "k_decoders_tc": "k3_decoders", "k_lbs": "k4_fk_lbs"}


def rows(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        return []
    hdr, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for name, metric, _ in KEYS:
            hits = [j for j, h in enumerate(hdr) if h == metric or h.endswith("." + metric)]
            if hits:
                i = hits[0]
                try:
                    v = float(row[i].replace(",", ""))
                except ValueError:
                    continue
                d[name] = v * UNIT.get(units[i], 1.0)
        res.append(d)
    return res


def main(argv):
    traffic_out = None
    if argv and argv[0] == "--traffic":
        traffic_out, argv = argv[1], argv[2:]
    allr = []
    for rep in argv:
        for d in rows(rep):
            d["report"] = rep.split("/")[-1]
            allr.append(d)
    if traffic_out:
        tr = {}
        for d in allr:
            st = STAGE.get(d["kernel"].split("<")[0])
            if "_c3" in d["report"] or "_c4" in d["report"]:
                continue  # microbench captures: not the C2 step's launches
            if st and "dram_read_B" in d:
                tr.setdefault(st, {"kernel": d["kernel"], "report": d["report"],
                                   "dram_bytes_per_launch": d["dram_read_B"] + d.get("dram_write_B", 0.0)})
        with open(traffic_out, "w") as fh:
            json.dump(tr, fh, indent=1)
        return
    cols = ["kernel", "report", "grid", "block", "regs", "time_us", "dram_read_B", "dram_write_B", "dram_pct",
            "tensor_pct", "sm_pct", "occupancy_pct"]
    print("| " + " | ".join(cols) + " |")
    print("|" + "---|" * len(cols))
    for d in allr:
        cells = []
        for c in cols:
            v = d.get(c, "")
            if isinstance(v, float):
                v = ("%.0f" % v) if abs(v) >= 100 else ("%.3g" % v)
            cells.append(str(v))
        print("| " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(sys.argv[1:])
