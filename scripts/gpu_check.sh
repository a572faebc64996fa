#!/bin/bash
# One GPU round trip: parity tests, conv + resnet bench lines, the 1-GPU scaling probe and the
# per-layer launch list of the batch-256 forward (ncu, after the plain runs exited 0).
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_rc=$? >> gpurun_out/gputests.log
tail -2 gpurun_out/gputests.log
timeout 300 python bench.py --workload conv --no-cpu-baseline > gpurun_out/bench_conv.json 2>gpurun_out/bench_conv.err
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_resnet.json 2>gpurun_out/bench_resnet.err
timeout 300 python scripts/scaling_probe.py > gpurun_out/scaling.txt 2>&1
if [ "$1" == "layers" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/launches_b256.csv python scripts/profile_resnet.py 256 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/launches_b32.csv python scripts/profile_resnet.py 32 1 > /dev/null 2>&1
fi
python - <<'PY'
import json
for f in ['bench_conv','bench_resnet']:
    try:
        d=json.load(open('gpurun_out/%s.json'%f)); print(f, d['value'], d['ms_per_step'], d['roofline']['achieved'])
    except Exception as e: print(f, 'FAILED', e)
PY
cat gpurun_out/scaling.txt
