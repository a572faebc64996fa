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
# DRAM traffic of one 256-image forward (roofline.traffic) and full captures of three real-data
# layers (3x3 s2b0.c2, residual K=64 s0b1.c3, residual K=256 s2b1.c3)
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file $O/traffic.csv python scripts/profile_resnet.py 256 1 > /dev/null 2>&1
python scripts/traffic_c3.py $O/traffic.csv > $O/traffic_c3_forward.json 2>&1; rm -f $O/traffic.csv
for i in 26 7 30; do
  timeout 900 ncu --set full --profile-from-start off -k regex:lut_p4w --launch-skip $i --launch-count 1 -o /tmp/fm_l$i python scripts/prof_net_layer.py > /dev/null 2>&1
  ncu -i /tmp/fm_l$i.ncu-rep --page raw --csv > $O/ncu_net_l$i.csv 2>/dev/null
  python scripts/ncu_summary.py $O/ncu_net_l$i.csv > $O/ncu_net_l${i}_summary.json 2>&1
done
for f in $O/bench_*_final.json $O/ref_resnet_final.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f'.split('/')[-1], d.get('value'), d.get('ms_per_step'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('clocks') or {}).get('reasons'))" 2>&1 | tail -1; done
grep predicted $O/scaling_probe_p4w.txt | tail -4
tail -3 $O/resnet_layers_b256_p4w.txt | head -1
