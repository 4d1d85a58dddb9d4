#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in 9 10 12 13; do ZERO_ADAM_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "config1_sim4 or single_rank or ragged" > gpurun_out/pytest_tma_$v.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tma_$v.log; done
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1500 python scripts/sweep.py --adam 5,9,10,11,12,13 --flat 2x4,4x4,8x4,2x8,4x8,8x8 --base ZERO_ADAM_VARIANT=5 > gpurun_out/sweep3.jsonl 2> gpurun_out/sweep3.err
