"""Summarise an ncu launch list (--metrics gpu__time_duration.sum[,dram__...]
--csv): one line per launch with kernel, grid, duration (us) and, when
captured, DRAM bytes read/written (MB)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
launches = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        key = (d["ID"], d.get("Process ID", ""))
        e = launches.setdefault(key, {"name": d["Kernel Name"], "grid": d["Grid Size"]})
        e[d["Metric Name"]] = (float(d["Metric Value"].replace(",", "")), d["Metric Unit"])

def scaled(v, unit, to):
    f = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3,
         "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
    return v * f.get(unit, float("nan"))

total = 0.0
for (i, _), e in launches.items():
    name = e["name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    name = name.replace("unnamed>::", "")
    t = e.get("gpu__time_duration.sum")
    us = scaled(*t, "us") if t else float("nan")
    total += us if us == us else 0
    line = f"{i:>4} {name[-44:]:<44} {e['grid']:>14} {us:10.1f} us"
    if "dram__bytes_read.sum" in e:
        line += f"  rd {scaled(*e['dram__bytes_read.sum'], 'MB'):10.1f} MB"
        line += f"  wr {scaled(*e['dram__bytes_write.sum'], 'MB'):8.1f} MB"
    print(line)
print(f"total kernel time {total / 1e3:.3f} ms over {len(launches)} launches")
