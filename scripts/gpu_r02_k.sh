#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
: > gpurun_out/mlp_k.jsonl
for i in 1 2; do
for c in 0 148 296; do
ZERO_STEP_SMALL_CTAS=$c timeout 300 python bench.py --config mlp1m --no-cpu-baseline --no-e2e --no-fp16-key | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'ctas': $c, 'us': d['ms_per_step']*1e3, 'launches': d['gpu_launches']/d['steps']}))" >> gpurun_out/mlp_k.jsonl
done
ZERO_STEP_SMALL=0 timeout 300 python bench.py --config mlp1m --no-cpu-baseline --no-e2e --no-fp16-key | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'ctas': 'off', 'us': d['ms_per_step']*1e3, 'launches': d['gpu_launches']/d['steps']}))" >> gpurun_out/mlp_k.jsonl
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/mlp_k_launches.csv \
   python bench.py --config mlp1m --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-fp16-key > /dev/null 2>&1
