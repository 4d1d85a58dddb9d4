#!/bin/bash
# One GPU session (run under gpurun): build, smoke, GPU tests, the default bench line (7.5B,
# stage 2, + fp16 key), the reference arm, every config at N = 1, and the round-2 ncu evidence.
# Outputs in gpurun_out/.
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/host_cpu.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
if [ "${CONFIGS:-0}" = "1" ]; then bash scripts/gpu_configs.sh; fi
if [ "${PROFILE:-0}" = "1" ]; then bash scripts/profile_r02.sh; fi
