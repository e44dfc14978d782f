"""Summarise an ncu --csv launch list: launches, mean us per kernel name."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    hdr, agg = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            agg.setdefault(d["Kernel Name"][:80], []).append(float(d["Metric Value"]))
    print(path)
    for k, v in agg.items():
        print(f"  {len(v):4d} {sum(v) / len(v) / 1000:9.1f} us  {k}")
