"""Key numbers of an `ncu --page raw --csv` export of one kernel capture: duration, issue, pipes,
shared-memory wavefronts (actual vs ideal: the bank-conflict replay factor), L1 / DRAM traffic
and the top stall reasons.  Usage: ncu_summary.py raw.csv [lookups_in_the_launch]."""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr, units, vals = rows[h], rows[h + 1], rows[h + 2]
d = {k: v for k, v in zip(hdr, vals)}
u = {k: v for k, v in zip(hdr, units)}
SCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1.0, "ms": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,                # -> bytes
         "hz": 1e-6, "Khz": 1e-3, "Mhz": 1.0, "Ghz": 1e3}                      # -> MHz


def f(k):
    try:
        return float(d[k].replace(",", "")) * SCALE.get(u.get(k, ""), 1.0)
    except (KeyError, ValueError):
        return None


out = {"kernel": d.get("Kernel Name", "")[:80],
       "duration_us": f("gpu__time_duration.sum"),
       "sm_mhz": f("sm__cycles_elapsed.avg.per_second"),
       "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
       "alu_pipe_pct": f("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
       "fma_pipe_pct": f("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
       "l1_wavefronts_pct": f("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
       "shared_ld_wavefronts": f("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"),
       "shared_wavefronts_ideal": f("memory_l1_wavefronts_shared_ideal"),
       "shared_wavefronts": f("memory_l1_wavefronts_shared"),
       "shared_ld_instructions": f("smsp__sass_inst_executed_op_shared_ld.sum"),
       "dram_bytes": (f("dram__bytes_read.sum") or 0) + (f("dram__bytes_write.sum") or 0),
       "registers": f("launch__registers_per_thread")}
if out["shared_wavefronts"] and out["shared_wavefronts_ideal"]:
    out["replay_factor"] = round(out["shared_wavefronts"] / out["shared_wavefronts_ideal"], 3)
if len(sys.argv) > 2 and out["duration_us"]:
    lk = float(sys.argv[2])
    out["lookups"] = lk
    out["T_lookups_per_s"] = round(lk / out["duration_us"] / 1e6, 3)   # lookups per us / 1e6 = T/s
    if out["shared_ld_wavefronts"]:
        out["lookups_per_shared_wavefront"] = round(lk / out["shared_ld_wavefronts"], 1)
stalls = {k.split("smsp__average_warps_issue_stalled_")[1].split("_per_issue_active")[0]: f(k)
          for k in hdr if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")}
out["top_stalls"] = dict(sorted(((k, round(v, 3)) for k, v in stalls.items() if v), key=lambda x: -x[1])[:6])
print(json.dumps(out, indent=1))
