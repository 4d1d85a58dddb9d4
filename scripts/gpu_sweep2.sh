#!/bin/bash
# Variant A/B on one box: parity of the candidate Adam (ZERO_ADAM_VARIANT) and flatten
# (ZERO_FLAT_TMA) variants through the C ABI, then the bench step under each (interleaved, repeated)
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
PT="tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py"
for v in ${ADAM_PAR:-}; do
  ZERO_ADAM_VARIANT=$v timeout 600 python -m pytest $PT -m gpu -q -x > gpurun_out/par_adam_$v.log 2>&1; echo "rc=$?" >> gpurun_out/par_adam_$v.log
done
for v in ${FLAT_PAR:-}; do
  ZERO_FLAT_TMA=$v timeout 600 python -m pytest $PT -m gpu -q -x > gpurun_out/par_flat_$v.log 2>&1; echo "rc=$?" >> gpurun_out/par_flat_$v.log
done
for i in 1 2 3; do
  timeout 900 python scripts/sweep.py --adam "${ADAM_SWEEP:-}" --flat-tma "${FLAT_SWEEP:-}" > gpurun_out/sweep2_$i.jsonl 2>&1
done
