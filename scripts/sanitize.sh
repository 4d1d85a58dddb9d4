#!/bin/bash
# compute-sanitizer over the small-size GPU parity tests (SURVEY §4 tier T5): every kernel of
# the step (k_flatten incl. the batched small-bucket launch and the fused N_d=1 decision path,
# k_flatten_wide via R32 over a 1-rank NCCL communicator, k_reduce_scatter default + variants,
# k_decide_*, k_adam_tma_st and the register k_adam, k_copy incl. P_a, k_load)
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/sanitize
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
SEL="ragged or clipping or bucket_order or stage3_gather or (single_rank and bf16) or (config1_sim4 and bf16 and R16)"
VAR="(variant_matches_oracle and (rs_plain_u2 or adam_tma or rs_grid_combine or rs_w16 or step_small)) or batching or step_record"
PA="round_trip and (100003 or 197) or backward_layer_order or call_order"
NC="r32_one_rank and bf16"
for tool in memcheck racecheck synccheck initcheck; do
  O=gpurun_out/sanitize/$tool
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --error-exitcode 17 --print-limit 20 \
     python -m pytest tests/test_gpu_parity.py -q -x -k "$SEL" -p no:cacheprovider > ${O}_parity.log 2>&1
  echo "rc=$?" >> ${O}_parity.log
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --error-exitcode 17 --print-limit 20 \
     python -m pytest tests/test_gpu_variants.py -q -x -k "$VAR" -p no:cacheprovider > ${O}_variants.log 2>&1
  echo "rc=$?" >> ${O}_variants.log
  timeout 900 compute-sanitizer --tool $tool --target-processes all --error-exitcode 17 --print-limit 20 \
     python -m pytest tests/test_gpu_activation.py -q -x -k "$PA" -p no:cacheprovider > ${O}_pa.log 2>&1
  echo "rc=$?" >> ${O}_pa.log
  timeout 900 compute-sanitizer --tool $tool --target-processes all --error-exitcode 17 --print-limit 20 \
     python -m pytest tests/test_gpu_nccl1.py -q -x -k "$NC" -p no:cacheprovider > ${O}_nccl.log 2>&1
  echo "rc=$?" >> ${O}_nccl.log
done
