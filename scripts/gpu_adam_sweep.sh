#!/bin/bash
# Adam variant A/B on one box: parity of the candidate variants through the C ABI, then
# the bench step under each variant (interleaved, repeated: clocks drift under the power cap)
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in ${VARIANTS:-21 22 23 24}; do
  ZERO_ADAM_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py -m gpu -q -x \
      > gpurun_out/adam_parity_$v.log 2>&1; echo "rc=$?" >> gpurun_out/adam_parity_$v.log
done
for i in 1 2 3; do
  timeout 900 python scripts/sweep.py --adam "11,${SWEEP:-21,22,23,24}" > gpurun_out/adam_sweep_$i.jsonl 2>&1
done
