#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_torch_zero.py -q -x > gpurun_out/pytest_torch_zero.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_torch_zero.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
