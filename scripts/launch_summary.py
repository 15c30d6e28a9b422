"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ik, iv, im, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name"), hdr.index("Metric Unit")
agg = OrderedDict()
for r in rows[h + 1:]:
    if len(r) > iv and r[im] == "gpu__time_duration.sum":
        v = float(r[iv].replace(",", ""))
        v = v / 1e3 if r[iu] in ("ns", "nsecond") else (v * 1e3 if r[iu] in ("ms", "msecond") else v)
        k = r[ik].split("(")[0][:70]
        agg.setdefault(k, []).append(v)
step = {k: v for k, v in agg.items() if any(s in k for s in ("tour_prep", "split_sweep", "split_finish"))}
tot = sum(sum(v) / len(v) for v in step.values())
print("%-72s %6s %10s %8s" % ("kernel", "count", "mean_us", "share"))
for k, v in agg.items():
    m = sum(v) / len(v)
    share = ("%.1f%%" % (100 * m / tot)) if k in step else "-"
    print("%-72s %6d %10.2f %8s" % (k, len(v), m, share))
print("step kernels (prep + sweep + finish) mean total: %.2f us (ncu: serialised, cold-cache)" % tot)
