#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + full capture of the top kernels.
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/host_cpu.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_adam -s 3 -c 1 -o gpurun_out/prof_adam \
    python bench.py --config gpt2_1.5b_l8 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_adam.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_flatten -s 40 -c 1 -o gpurun_out/prof_flatten \
    python bench.py --config gpt2_1.5b_l8 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_flatten.log 2>&1
ls -la gpurun_out
