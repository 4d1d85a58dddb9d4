#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config mlp1m --no-cpu-baseline --no-e2e --no-fp16-key > gpurun_out/mlp_eager.json 2> gpurun_out/mlp.err
timeout 300 python bench.py --config mlp1m --graph --no-cpu-baseline --no-e2e > gpurun_out/mlp_graph.json 2>> gpurun_out/mlp.err
bash scripts/gpu_rs_sweep.sh
timeout 1200 python scripts/max_model.py --device > gpurun_out/max_model_device.jsonl 2> gpurun_out/max_model_device.err
