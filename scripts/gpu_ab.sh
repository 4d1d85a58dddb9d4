#!/bin/bash
# A/B on one box: the current build vs an alternative build of the same ABI (ZERO_LIB_PATH),
# the default bench step, interleaved and repeated; plus the GPU parity subset on the current build
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
ALT=${ALT:-paper_1910_02054_b200/libzero_b200_alt.so}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py tests/test_gpu_edge.py tests/test_gpu_graph.py -m gpu -q -x > gpurun_out/ab_parity.log 2>&1; echo "rc=$?" >> gpurun_out/ab_parity.log
for i in 1 2 3; do
  timeout 600 python scripts/sweep.py --adam 21 ${SWEEP_ARGS:-} > gpurun_out/ab_cur_$i.jsonl 2>&1
  ZERO_LIB_PATH=$PWD/$ALT timeout 600 python scripts/sweep.py --adam 21 ${SWEEP_ARGS:-} > gpurun_out/ab_alt_$i.jsonl 2>&1
done
