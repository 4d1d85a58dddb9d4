#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in 1 2 3 4; do ZERO_FLAT_TMA=$v timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "single_rank or ragged or clipping" > gpurun_out/pytest_ftma_$v.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ftma_$v.log; done
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1500 python scripts/sweep.py --adam 11,14,15,16,17,18 --flat-tma 1,2,3,4 > gpurun_out/sweep4.jsonl 2> gpurun_out/sweep4.err
