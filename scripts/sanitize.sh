#!/bin/bash
# compute-sanitizer over the small-size GPU parity tests (SURVEY §4 tier T5)
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
SEL="ragged or clipping or bucket_order or stage3_gather or (single_rank and bf16) or (config1_sim4 and bf16 and R16)"
PA="round_trip and (100003 or 197) or backward_layer_order or call_order"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --error-exitcode 17 --print-limit 20 \
     python -m pytest tests/test_gpu_parity.py -q -x -k "$SEL" -p no:cacheprovider > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
  timeout 900 compute-sanitizer --tool $tool --target-processes all --error-exitcode 17 --print-limit 20 \
     python -m pytest tests/test_gpu_activation.py -q -x -k "$PA" -p no:cacheprovider > gpurun_out/sanitize_pa_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_pa_$tool.log
done
