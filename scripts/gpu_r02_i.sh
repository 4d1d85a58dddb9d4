#!/bin/bash
# N>1 flows end to end on one GPU (ranks time-slice it: functional, not throughput)
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ipc.py -q -k "share_one_gpu" > gpurun_out/pytest_ipc8.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ipc8.log
: > gpurun_out/bench_same_dev.jsonl
for spec in "8 2" "8 3" "4 1" "2 0"; do
  set -- $spec
  ZERO_BENCH_SAME_DEVICE=1 timeout 900 python bench.py --gpus $1 --stage $2 --config gpt2_1.5b_l8 --steps 3 --warmup 3 \
      --no-cpu-baseline --no-fp16-key --e2e-steps 2 >> gpurun_out/bench_same_dev.jsonl 2>> gpurun_out/bench_same_dev.err
  echo "n=$1 stage=$2 rc=$?" >> gpurun_out/bench_same_dev.err
done
ZERO_BENCH_SAME_DEVICE=1 timeout 600 python scripts/collective_sweep.py --gpus 2 --min-mb 16 --max-mb 64 --iters 3 --warmup 2 > gpurun_out/collective_same_dev.jsonl 2> gpurun_out/collective_same_dev.err
echo "sweep rc=$?" >> gpurun_out/collective_same_dev.err
