#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python scripts/sweep.py --adam "" --flat 4x4,8x4,4x2,8x2,2x4 > gpurun_out/sweep6.jsonl 2> gpurun_out/sweep6.err
ZERO_FLAT_STREAMS=1 timeout 600 python bench.py --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/bench_1stream.json 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
