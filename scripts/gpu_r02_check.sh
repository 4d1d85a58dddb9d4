#!/bin/bash
# Round-2 check on one B200: build, GPU tests, smoke, the default bench line (7.5B, stage 2),
# the reference arm, and the N>1 flow with 2 ranks sharing cuda:0 (functional).
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ZERO_BENCH_SAME_DEVICE=1 timeout 600 python bench.py --gpus 2 --config gpt2_1.5b --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n2_same.json 2> gpurun_out/bench_n2_same.err; echo "rc=$?" >> gpurun_out/bench_n2_same.err
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
