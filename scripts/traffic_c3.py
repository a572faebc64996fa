"""Sum the DRAM traffic of one ResNet-50 (c3) forward from an ncu launch list of
scripts/profile_resnet.py taken with --metrics dram__bytes_read.sum,dram__bytes_write.sum,
gpu__time_duration.sum: the forward is everything after the last input quantize launch.
Prints a JSON summary (bytes per forward for the LUT kernels and for all kernels)."""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[h]
ki, mi, vi, ui, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "usecond": 1e3,
         "nsecond": 1, "ms": 1e6, "msecond": 1e6}
launch = collections.OrderedDict()
for r in rows[h + 1:]:
    if len(r) <= vi:
        continue
    d = launch.setdefault(r[ii], {"name": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
L = list(launch.values())
start = [i for i, d in enumerate(L) if "quantize_nchw_to_nhwc" in d["name"]][-1]
fw = L[start:]
lut = [d for d in fw if any(k in d["name"] for k in ("lut_p4w", "lut_mm", "p4_pack_tables", "lut_p4_kernel"))]


def tot(ds, k):
    return int(sum(d.get(k, 0) for d in ds))


out = {"launches_forward": len(fw), "lut_launches": len(lut),
       "lut_dram_read_bytes": tot(lut, "dram__bytes_read.sum"),
       "lut_dram_write_bytes": tot(lut, "dram__bytes_write.sum"),
       "all_dram_bytes": tot(fw, "dram__bytes_read.sum") + tot(fw, "dram__bytes_write.sum"),
       "lut_time_ns": tot(lut, "gpu__time_duration.sum"), "all_time_ns": tot(fw, "gpu__time_duration.sum")}
out["lut_dram_bytes"] = out["lut_dram_read_bytes"] + out["lut_dram_write_bytes"]
print(json.dumps(out, indent=1))
