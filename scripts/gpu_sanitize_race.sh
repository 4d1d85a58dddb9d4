#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --error-exitcode 17 --print-limit 10 \
   python -m pytest tests/test_gpu_parity.py -q -x -k "single_rank and bf16 and (0 or 1)" -p no:cacheprovider > gpurun_out/sanitize_racecheck.log 2>&1
echo "rc=$?" >> gpurun_out/sanitize_racecheck.log
timeout 600 python scripts/sweep.py --adam 11 > gpurun_out/sweep_fence.jsonl 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
