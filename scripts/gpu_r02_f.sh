#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config mlp1m --no-cpu-baseline --no-e2e --no-fp16-key > gpurun_out/mlp_eager.json 2> gpurun_out/mlp.err
timeout 300 python bench.py --config mlp1m --graph --no-cpu-baseline --no-e2e > gpurun_out/mlp_graph.json 2>> gpurun_out/mlp.err
rm -rf gpurun_out/rs_sweep
RS_RANKS="4 8" bash scripts/gpu_rs_sweep.sh
timeout 600 python scripts/sim_bench.py --ranks 4 --stage 2 > gpurun_out/sim_step.jsonl 2>&1
timeout 1200 python scripts/max_model.py --device > gpurun_out/max_model_device.jsonl 2> gpurun_out/max_model_device.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
