"""Match an ncu launch list of scripts/profile_resnet.py to the ResNet layers (per-layer
time and fraction of the 32-lookups/clk/SM roofline at 1965 MHz)."""
import collections
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_04071_b200.resnet import _out, layer_specs  # noqa: E402

path = sys.argv[1]
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
rows = list(csv.reader(open(path)))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[h]
ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
launch = collections.OrderedDict()
for r in rows[h + 1:]:
    d = launch.setdefault(r[ii], {"name": r[ki]})
    d[r[mi]] = r[vi]
L = list(launch.values())
start = [i for i, d in enumerate(L) if "quantize_nchw_to_nhwc" in d["name"]][-1]
fw = L[start:]
sp = {s[0]: s for s in layer_specs()}


def conv(name, hi, wi):
    _, _, cout, cin, k, s, p = sp[name]
    ho, wo = _out(hi, k, s, p), _out(wi, k, s, p)
    return ho, wo, (name, batch * ho * wo * cout * cin * k * k, (batch * ho * wo, cout, cin * k * k))


order = []
ho, wo, e = conv("stem", 224, 224)
order.append(e)
h, w = _out(ho, 3, 2, 1), _out(wo, 3, 2, 1)
for b in [s[0][:-3] for s in layer_specs() if s[0].endswith(".c1")]:
    if b + ".down" in sp:
        order.append(conv(b + ".down", h, w)[2])
    h1, w1, e = conv(b + ".c1", h, w); order.append(e)
    h2, w2, e = conv(b + ".c2", h1, w1); order.append(e)
    h, w, e = conv(b + ".c3", h2, w2); order.append(e)
order.append(("fc", batch * 1000 * 2048, (batch, 1000, 2048)))
luts = [d for d in fw if ("lut_mm" in d["name"] or "lut_p4" in d["name"])]
tot = totl = 0.0
for (n, lk, mnk), d in zip(order, luts):
    t = float(d["gpu__time_duration.sum"]) / 1e3
    tot += t
    totl += lk
    print("%-11s M=%7d N=%5d K=%5d %-3s grid=%-6s %8.1f us %6.0f Glk/s frac %.2f" % (
        n, *mnk, "p4" if "lut_p4" in d["name"] else "v1", d.get("launch__grid_size", "?"), t,
        lk / t / 1e3, lk / t / 1e3 / 9306.24))
print("LUT kernels: %.2f ms, %.0f Glk/s, frac %.3f" % (tot / 1e3, totl / tot / 1e3, totl / tot / 1e3 / 9306.24))
for d in fw:
    if "lut_mm" not in d["name"] and "lut_p4" not in d["name"]:
        print("  %-60s %8.1f us" % (d["name"][:60], float(d["gpu__time_duration.sum"]) / 1e3))
