#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in 5 6 7 8; do ZERO_ADAM_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "config1_sim4 or single_rank" > gpurun_out/pytest_tma_$v.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tma_$v.log; done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
timeout 1200 python scripts/sweep.py --adam 1,5,6,7,8 --base ZERO_FLAT_VECS=4,ZERO_FLAT_CTAS=4 > gpurun_out/sweep2.jsonl 2> gpurun_out/sweep2.err
