"""Hottest SASS instructions of an ncu report (source page, sass view).

    python tools/sass_hot.py report.ncu-rep [n] [sort_key]
sort_key: a column of the source page, default "Warp Stall Sampling (All Samples)".
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
key = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
out = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
hi = next(i for i, x in enumerate(r) if x and x[0] == "Address")
h = r[hi]
rows = [x for x in r[hi + 1:] if len(x) == len(h)]


def f(x, k):
    try:
        return float(x[h.index(k)].replace(",", ""))
    except (ValueError, IndexError):
        return 0.0


tot = sum(f(x, key) for x in rows) or 1.0
cols = ["L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal", "Instructions Executed"]
print("%% of %s | addr | %s | sass" % (key, " | ".join(cols)))
for x in sorted(rows, key=lambda x: -f(x, key))[:n]:
    print("%5.1f%% %s %s  %s" % (100 * f(x, key) / tot, x[0], " ".join("%9.0f" % f(x, c) for c in cols),
                                 x[1][:80]))
print("total L1 wavefronts shared %.0f (ideal %.0f)" % (sum(f(x, cols[0]) for x in rows),
                                                        sum(f(x, cols[1]) for x in rows)))
