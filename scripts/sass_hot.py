"""Summarise an `ncu --page source --csv --print-source sass` export: instruction share by
execution frequency (per-stage / per-tile groups) and the lines with the most stall samples."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
which = int(sys.argv[2]) if len(sys.argv) > 2 else 0
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif r and r[0] == "Address":
        cur["hdr"] = r
    elif cur is not None and "hdr" in cur and len(r) == len(cur["hdr"]):
        cur["rows"].append(dict(zip(cur["hdr"], r)))
print(len(blocks), "kernels")
B = blocks[which]
R = B["rows"]
f = lambda r, k: float(r[k] or 0)
tot = sum(f(r, "Instructions Executed") for r in R)
tots = sum(f(r, "Warp Stall Sampling (All Samples)") for r in R)
c, n, sm = collections.Counter(), collections.Counter(), collections.Counter()
for r in R:
    e = int(f(r, "Instructions Executed"))
    c[e] += e; n[e] += 1; sm[e] += f(r, "Warp Stall Sampling (All Samples)")
print(B["name"], "inst", tot, "samples", tots)
for e, v in c.most_common(12):
    print("exec %10d lines %5d inst-share %.3f samp-share %.3f" % (e, n[e], v / tot, sm[e] / tots))
for r in sorted(R, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]:
    print("%6d %10d %s %s" % (f(r, "Warp Stall Sampling (All Samples)"), f(r, "Instructions Executed"), r["Address"][-5:], r["Source"][:70]))
