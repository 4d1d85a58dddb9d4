#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 300 python bench.py --stage 3 --steps 30 --no-e2e --no-cpu-baseline > gpurun_out/bench_s3.json 2> gpurun_out/bench_s3.err
ZERO_BENCH_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
   bench.py --gpus 2 --config gpt2_1.5b_l8 --stage 3 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_n2_s3.json 2> gpurun_out/bench_n2_s3.err
echo "rc=$?" >> gpurun_out/bench_n2_s3.err
