#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_ipc.py -q -k overlap > gpurun_out/pytest_overlap.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_overlap.log
timeout 300 python bench.py --config mlp1m --no-cpu-baseline --no-e2e --no-fp16-key > gpurun_out/mlp_eager.json 2> gpurun_out/mlp.err
timeout 300 python bench.py --config mlp1m --no-cpu-baseline --no-e2e --no-fp16-key --phase-events on > gpurun_out/mlp_eager_ev.json 2>> gpurun_out/mlp.err
timeout 300 python bench.py --config mlp1m --graph --no-cpu-baseline --no-e2e > gpurun_out/mlp_graph.json 2>> gpurun_out/mlp.err
rm -f gpurun_out/rs_sweep/*
bash scripts/gpu_rs_sweep.sh
timeout 1200 python scripts/max_model.py --device > gpurun_out/max_model_device.jsonl 2> gpurun_out/max_model_device.err
