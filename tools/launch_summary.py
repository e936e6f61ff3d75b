"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
one line per launch, kernel name, grid, duration in microseconds."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        print(f'{d["ID"]:>4} {name[-48:]:<48} {d["Grid Size"]:>16} {float(d["Metric Value"]) / 1e3:10.1f} us')
