"""Per-launch table of an ncu --csv metrics log: `python tools/launch_table.py file.csv`.
Prints one line per launch (kernel, metrics) and the summed duration."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
launches = OrderedDict()
for r in rows[h + 1:]:
    if len(r) > vi:
        launches.setdefault(r[ii], {"kernel": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
tot = 0.0
for i, d in launches.items():
    t = d.get("gpu__time_duration.sum", 0.0)
    tot += t
    extra = " ".join(f"{k.split('__')[1].split('.')[0]}={v / 1e6:.1f}MB" for k, v in d.items() if k.startswith("dram"))
    print(f"{i:>4} {t / 1e3:8.1f} us  {d['kernel'][:70]}  {extra}")
print(f"sum {tot / 1e3:.1f} us over {len(launches)} launches")
