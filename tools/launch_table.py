"""Per-kernel table of an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
d = collections.OrderedDict()
for r in rows[1:]:
    d.setdefault(r[ki][:70], []).append(float(r[vi].replace(",", "")) / 1000)
for k, v in d.items():
    print("%3d  %9.1f us  %s" % (len(v), sum(v), k))
