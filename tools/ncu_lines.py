"""Map an ncu report's per-SASS warp-stall samples to CUDA source lines via
nvdisasm line info of the matching cubin (the report's function must come
from that cubin's build).

    python tools/ncu_lines.py report.ncu-rep build/obj/k_transformer_tc.o FUNC_MANGLED [N]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def main():
    rep, obj, fn = sys.argv[1:4]
    n = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    ci = h.index("Warp Stall Sampling (All Samples)")
    body = [r for r in rows[2:] if len(r) > ci]
    base = int(body[0][0], 16)
    samp = {int(r[0], 16) - base: float(r[ci] or 0) for r in body}
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
        cub = [os.path.join(d, f) for f in os.listdir(d) if f.endswith(".cubin")][0]
        dis = subprocess.run(["nvdisasm", "--print-line-info", cub], capture_output=True, text=True).stdout
    loc, on, off2loc = None, False, {}
    for line in dis.split("\n"):
        if line.startswith("//----") and ".text." in line:
            on = (".text." + fn) in line
            continue
        if not on:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            loc = (m.group(1), int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", line)
        if m:
            off2loc[int(m.group(1), 16)] = loc
    agg = collections.Counter()
    for off, v in samp.items():
        agg[off2loc.get(off)] += v
    tot = sum(samp.values()) or 1.0
    cache = {}
    for l, v in agg.most_common(n):
        txt = ""
        if l:
            if l[0] not in cache:
                try:
                    cache[l[0]] = open(l[0]).read().split("\n")
                except OSError:
                    cache[l[0]] = []
            src = cache[l[0]]
            txt = src[l[1] - 1].strip()[:90] if l[1] - 1 < len(src) else ""
        name = "%s:%d" % (os.path.basename(l[0]), l[1]) if l else "?"
        print("%5.1f %-28s %s" % (100 * v / tot, name, txt))


if __name__ == "__main__":
    main()
