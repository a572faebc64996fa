#!/bin/bash
# GPU round trip for the int32 tables: their parity tests (L1 gather and SM-resident halves),
# bench lines of c2 with a +-1e5 ACU in both forms, the whole GPU suite, smoke(), the default
# bench, and the ncu launch list + one full capture of each int32 form (after plain runs exit 0).
cd "$(dirname "$0")/.."
timeout 400 python -m pytest tests/test_gpu_i32.py -x -q > gpurun_out/i32tests.log 2>&1; echo rc=$? >> gpurun_out/i32tests.log
tail -3 gpurun_out/i32tests.log
for r in 0 1; do
AXQ_I32_RESIDENT=$r timeout 300 python bench.py --workload conv --lut err1e5 --no-cpu-baseline > gpurun_out/bench_conv_i32_r$r.json 2>gpurun_out/bench_conv_i32_r$r.err; echo conv_i32 r$r rc=$?
done
python - <<'PY'
import json
for f in ['bench_conv_i32_r0','bench_conv_i32_r1']:
    try:
        d=json.load(open('gpurun_out/%s.json'%f)); print(f, d['value'], d['ms_per_step'], d['roofline'].get('achieved'), d['metric_roofline']['frac'] if 'metric_roofline' in d else d['roofline'].get('metric_roofline',{}).get('frac'))
    except Exception as e: print(f, 'FAILED', e)
PY
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_rc=$? >> gpurun_out/gputests.log
tail -3 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_resnet.json 2>gpurun_out/bench_resnet.err
python -c "import json; d=json.load(open('gpurun_out/bench_resnet.json')); print('resnet', d['value'], d['ms_per_step'], d['roofline']['frac'])"
for r in 0 1; do
AXQ_I32_RESIDENT=$r timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_conv_i32_r$r.csv python bench.py --workload conv --lut err1e5 --no-cpu-baseline --no-e2e --steps 1 --warmup 3 > /dev/null 2>&1; echo ncu_list r$r rc=$?
AXQ_I32_RESIDENT=$r timeout 600 ncu --set full --clock-control none --import-source on -k regex:lut_mm_kernel -s 3 -c 1 -o gpurun_out/ncu_conv_i32_r$r python bench.py --workload conv --lut err1e5 --no-cpu-baseline --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu_full_r$r.log 2>&1; echo ncu_full r$r rc=$?
done
