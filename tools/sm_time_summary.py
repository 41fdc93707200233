"""Summarise tools/sm_time.sh output: SM-microseconds per kernel for one batch
(second of the two repetitions), at the 1.965 GHz boost clock."""
import collections
import csv
import sys

rows = [r for r in csv.DictReader(line for line in open(sys.argv[1]) if not line.startswith("=="))]
k = collections.OrderedDict()
for r in rows:
    k.setdefault((r["ID"], r["Kernel Name"][:44]), {})[r["Metric Name"]] = r["Metric Value"]
items = list(k.items())
items = items[len(items) // 2:]
tot = 0.0
for (i, name), m in items:
    smus = float(m["sm__cycles_active.sum"]) / 1965.0
    tot += smus
    print("%-44s grid=%6s regs=%4s dur=%8.2fus SM-us=%8.1f" % (name, m["launch__grid_size"],
          m["launch__registers_per_thread"], float(m["gpu__time_duration.sum"]) / 1e3, smus))
print("total SM-us per batch %.1f  (/148 = %.2f us)" % (tot, tot / 148))
