"""Print an ncu --metrics gpu__time_duration.sum launch list (CSV) as (id, kernel, us, grid, block)
rows; optional [start, stop) range of launch ids."""
import csv
import sys


def rows(path):
    h = None
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            h = r
            continue
        if h and len(r) == len(h):
            d = dict(zip(h, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"]) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
                                                 "nsecond": 1e-3}.get(d["Metric Unit"], 1.0)
                yield int(d["ID"]), d["Kernel Name"], v, d.get("Grid Size"), d.get("Block Size")


if __name__ == "__main__":
    a = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    b = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 30
    for i, k, us, g, bl in rows(sys.argv[1]):
        if a <= i < b:
            print("%5d %9.2f us  %-16s %-12s %s" % (i, us, g, bl, k[:90]))
