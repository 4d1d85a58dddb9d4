#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvidia-smi --query-gpu=memory.used,memory.total --format=csv > gpurun_out/mem.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
timeout 900 python bench.py --config gpt_7.5b --steps 20 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/bench_7p5b.json 2> gpurun_out/bench_7p5b.err
