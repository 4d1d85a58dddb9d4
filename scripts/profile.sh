#!/bin/bash
# ncu evidence for the default kernels: launch list of the bench step + one full capture each
# of k_adam_tma and k_flatten on the 8-layer slice of the GPT-2 1.5B layout.
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_adam -s 3 -c 1 -o gpurun_out/prof_adam -f \
    python bench.py --config gpt2_1.5b_l8 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_adam.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_flatten -s 20 -c 1 -o gpurun_out/prof_flatten -f \
    python bench.py --config gpt2_1.5b_l8 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_flatten.log 2>&1
