#!/bin/bash
# build + GPU tests + a short sweep of the default configuration
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python scripts/sweep.py --adam "11,11" --flat "4x4,8x4" > gpurun_out/sweep_quick.jsonl 2> gpurun_out/sweep_quick.err
