#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_graph.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py -q > gpurun_out/pytest_l.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_l.log
: > gpurun_out/mlp_l.jsonl
for i in 1 2 3; do
for p in 1 0; do
ZERO_ADAM_PDL=$p timeout 300 python bench.py --config mlp1m --no-cpu-baseline --no-e2e --no-fp16-key | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'pdl': $p, 'graph': False, 'us': d['ms_per_step']*1e3}))" >> gpurun_out/mlp_l.jsonl
ZERO_ADAM_PDL=$p timeout 300 python bench.py --config mlp1m --graph --no-cpu-baseline --no-e2e | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'pdl': $p, 'graph': True, 'us': d['ms_per_step']*1e3}))" >> gpurun_out/mlp_l.jsonl
done
done
