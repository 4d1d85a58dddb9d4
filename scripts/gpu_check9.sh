#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
ZERO_BENCH_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
   bench.py --gpus 2 --config gpt2_1.5b_l8 --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/bench_n2_samedev.json 2> gpurun_out/bench_n2_samedev.err
echo "rc=$?" >> gpurun_out/bench_n2_samedev.err
ZERO_BENCH_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
   bench.py --gpus 2 --config gpt2_1.5b_l8 --stage 3 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_n2_s3.json 2> gpurun_out/bench_n2_s3.err
echo "rc=$?" >> gpurun_out/bench_n2_s3.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 \
   bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_ref_n2.json 2> gpurun_out/bench_ref_n2.err
echo "rc=$?" >> gpurun_out/bench_ref_n2.err
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
