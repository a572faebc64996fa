#!/bin/bash
# Bench line + ncu launch list + one full capture of the int32-table conv (--lut err1e5).
cd "$(dirname "$0")/.."
timeout 300 python bench.py --workload conv --lut err1e5 --no-cpu-baseline > gpurun_out/bench_conv_i32.json 2>gpurun_out/bench_conv_i32.err; echo conv_i32 rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_conv_i32.json')); print(d['value'], d['ms_per_step'], d['roofline'])"
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_conv_i32.csv python bench.py --workload conv --lut err1e5 --no-cpu-baseline --no-e2e --steps 1 --warmup 3 > /dev/null 2>&1; echo ncu_list rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lut_mm_kernel -s 3 -c 1 -o gpurun_out/ncu_conv_i32 python bench.py --workload conv --lut err1e5 --no-cpu-baseline --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu_full.log 2>&1; echo ncu_full rc=$?
