#!/bin/bash
# Same-box A/B: alternate runs of libaxq_base.so (A) and libaxq.so (B) on the ResNet bench
# and one conv layer; prints ms per step for each.
cd "$(dirname "$0")/.."
for i in 1 2; do
  for L in paper_2203_04071_b200/libaxq_base.so paper_2203_04071_b200/libaxq.so; do
    r=$(AXQ_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'])")
    c=$(AXQ_LIB=$L timeout 300 python scripts/prof_layer.py 256 56 56 64 256 1 1 1 5 2>/dev/null | tail -1)
    echo "$(basename $L) resnet_ms=$r  c3: $c"
  done
done
