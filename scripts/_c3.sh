cd $GRAFT_REPO_ROOT
run() { AXQ_P4W_MAIN_CW=$1 AXQ_P4W_MAIN_CW_MAX_K=$2 timeout 300 python bench.py --workload resnet --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/r.json 2>gpurun_out/r.err; python -c "import json,sys; d=json.load(open('gpurun_out/r.json')); print(d['ms_per_step'])" 2>/dev/null || (tail -2 gpurun_out/r.err | head -2); }
for i in 1 2; do for c in "28 0" "20 64" "20 128" "24 128" "20 256"; do set -- $c; echo "main=$1 maxk=$2 resnet $(run $1 $2)"; done; done > gpurun_out/sweep.txt
cat gpurun_out/sweep.txt
