#!/bin/bash
# A/B: the current build vs paper_1910_02054_b200/libzero_b200_head.so on the same box
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for i in 1 2; do
  timeout 600 python scripts/sweep.py --adam 11 > gpurun_out/ab_cur_$i.jsonl 2>&1
  ZERO_LIB_PATH=$PWD/paper_1910_02054_b200/libzero_b200_head.so timeout 600 python scripts/sweep.py --adam 11 > gpurun_out/ab_head_$i.jsonl 2>&1
done
