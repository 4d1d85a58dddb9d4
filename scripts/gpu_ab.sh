#!/bin/bash
# A/B: the current build vs an alternative build of the same ABI (ZERO_LIB_PATH) on the same box
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
ALT=${ALT:-paper_1910_02054_b200/libzero_b200_alt.so}
for i in 1 2; do
  timeout 600 python scripts/sweep.py --adam 11 > gpurun_out/ab_cur_$i.jsonl 2>&1
  ZERO_LIB_PATH=$PWD/$ALT timeout 600 python scripts/sweep.py --adam "" --flat "4x4,4x5,4x6" > gpurun_out/ab_alt_$i.jsonl 2>&1
done
