#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_ipc.py tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_graph.py -q > gpurun_out/pytest_sel.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sel.log
timeout 300 python bench.py --config mlp1m --no-cpu-baseline --no-e2e --no-fp16-key > gpurun_out/mlp_eager.json 2> gpurun_out/mlp.err
timeout 300 python bench.py --config mlp1m --graph --no-cpu-baseline --no-e2e > gpurun_out/mlp_graph.json 2>> gpurun_out/mlp.err
ZERO_ADAM_SMALL=0 timeout 300 python bench.py --config mlp1m --no-cpu-baseline --no-e2e --no-fp16-key > gpurun_out/mlp_eager_tma.json 2>> gpurun_out/mlp.err
ZERO_ADAM_SMALL=0 timeout 300 python bench.py --config mlp1m --graph --no-cpu-baseline --no-e2e > gpurun_out/mlp_graph_tma.json 2>> gpurun_out/mlp.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/mlp_launches.csv \
   python bench.py --config mlp1m --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-fp16-key > gpurun_out/mlp_ncu.log 2>&1
bash scripts/gpu_rs_sweep.sh
timeout 1200 python scripts/max_model.py --device > gpurun_out/max_model_device.jsonl 2> gpurun_out/max_model_device.err
