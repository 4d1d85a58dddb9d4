#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/mlp_j.jsonl
for i in 1 2; do
timeout 300 python bench.py --config mlp1m --no-cpu-baseline --no-e2e --no-fp16-key >> gpurun_out/mlp_j.jsonl 2>> gpurun_out/mlp.err
timeout 300 python bench.py --config mlp1m --graph --no-cpu-baseline --no-e2e >> gpurun_out/mlp_j.jsonl 2>> gpurun_out/mlp.err
ZERO_STEP_SMALL=0 timeout 300 python bench.py --config mlp1m --no-cpu-baseline --no-e2e --no-fp16-key >> gpurun_out/mlp_j.jsonl 2>> gpurun_out/mlp.err
done
