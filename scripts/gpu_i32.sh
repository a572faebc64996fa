#!/bin/bash
# GPU round trip for the SM-resident int32 table: its parity tests first, then the whole GPU
# suite, smoke(), bench lines (conv with the +-1e5 ACU, conv default, resnet) and the ncu
# launch list + one full capture of the int32-table conv (after the plain runs exited 0).
cd "$(dirname "$0")/.."
timeout 300 python -m pytest tests/test_gpu_i32.py -x -q > gpurun_out/i32tests.log 2>&1; echo rc=$? >> gpurun_out/i32tests.log
tail -3 gpurun_out/i32tests.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_rc=$? >> gpurun_out/gputests.log
tail -3 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 300 python bench.py --workload conv --lut err1e5 --no-cpu-baseline > gpurun_out/bench_conv_i32.json 2>gpurun_out/bench_conv_i32.err; echo conv_i32 rc=$?
timeout 300 python bench.py --workload conv --lut err2000 --no-cpu-baseline > gpurun_out/bench_conv16.json 2>gpurun_out/bench_conv16.err
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_resnet.json 2>gpurun_out/bench_resnet.err
python - <<'PY'
import json
for f in ['bench_conv_i32','bench_conv16','bench_resnet']:
    try:
        d=json.load(open('gpurun_out/%s.json'%f)); print(f, d['value'], d['ms_per_step'], d['roofline'].get('achieved'), d['roofline'].get('frac'))
    except Exception as e: print(f, 'FAILED', e)
PY
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_conv_i32.csv python bench.py --workload conv --lut err1e5 --no-cpu-baseline --no-e2e --steps 1 --warmup 3 > /dev/null 2>&1; echo ncu_list rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lut_mm_kernel -s 3 -c 1 -o gpurun_out/ncu_conv_i32 python bench.py --workload conv --lut err1e5 --no-cpu-baseline --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu_full.log 2>&1; echo ncu_full rc=$?
