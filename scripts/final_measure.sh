#!/bin/bash
# Round-end measurement set (one gpurun call): GPU parity tests, every bench workload, the
# ncu launch list of the default bench, per-layer tables at batch 256 / 32, the scaling probe.
cd "$(dirname "$0")/.."
O=gpurun_out/final; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/gputests.log 2>&1; tail -1 $O/gputests.log
timeout 600 python bench.py > $O/bench_resnet_final.json 2> $O/bench_resnet.err
timeout 600 python bench.py --quantizer paper --no-cpu-baseline > $O/bench_resnet_paper_final.json 2> $O/bench_resnet_paper.err
for w in conv linear lstm gemm; do timeout 600 python bench.py --workload $w > $O/bench_${w}_final.json 2> $O/bench_$w.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/ref_resnet_final.json 2> $O/ref.err
timeout 300 python scripts/scaling_probe.py > $O/scaling_probe_p4w.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $O/launches_bench_resnet.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $O/launches_b256.csv python scripts/profile_resnet.py 256 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $O/launches_b32.csv python scripts/profile_resnet.py 32 1 > /dev/null 2>&1
python scripts/layer_table.py $O/launches_b256.csv 256 > $O/resnet_layers_b256_p4w.txt 2>&1
python scripts/layer_table.py $O/launches_b32.csv 32 > $O/resnet_layers_b32_p4w.txt 2>&1
rm -f $O/launches_b256.csv $O/launches_b32.csv
for f in $O/bench_*_final.json $O/ref_resnet_final.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f'.split('/')[-1], d.get('value'), d.get('ms_per_step'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('clocks') or {}).get('reasons'))" 2>&1 | tail -1; done
grep predicted $O/scaling_probe_p4w.txt | tail -4
tail -3 $O/resnet_layers_b256_p4w.txt | head -1
