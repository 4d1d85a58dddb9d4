#!/bin/bash
# ncu evidence for the default kernels (run on the GPU box):
#  1. launch list of the bench step (every launch with its device time)
#  2. --set full capture of k_adam_tma in the bench's own launch configuration (GPT-2 1.5B, stage 1)
#  3. --set full capture of one k_flatten launch (a GPT-2 block bucket)
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_adam -s 3 -c 1 -o gpurun_out/prof_adam -f \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_adam.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_flatten -s 160 -c 1 -o gpurun_out/prof_flatten -f \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_flatten.log 2>&1
for r in prof_adam prof_flatten; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/$r.details.csv 2>/dev/null
done
