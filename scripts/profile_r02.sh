#!/bin/bash
# Round-2 ncu evidence (one GPU, gpurun):
#  1. launch list of the default bench step (7.5B layout, stage 2, N = 1)
#  2. --set full of the fused Adam and of one flatten launch in the bench's launch configuration
#     (GPT-2 1.5B, stage 1: the same kernels; at 7.5B ncu's replay would have to save ~120 GB)
#  3. --set full of one pull reduce-scatter (N_d = 4 simulated ranks, GPT-2 block bucket, stage 2)
#  4. --set full of one stage-3 layer-gather k_copy (N_d = 4 simulated ranks)
#  5. launch list of config 1 (1M-param MLP, stage 2, N = 1)
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/prof
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
O=gpurun_out/prof
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_7p5b.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-fp16-key > $O/launches_7p5b.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_adam -s 3 -c 1 -o $O/adam -f \
    python bench.py --config gpt2_1.5b --stage 1 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-fp16-key > $O/adam.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_flatten -s 160 -c 1 -o $O/flatten -f \
    python bench.py --config gpt2_1.5b --stage 1 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-fp16-key > $O/flatten.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_reduce_scatter -s 40 -c 1 -o $O/rs -f \
    python scripts/sim_bench.py --ranks 4 --stage 2 --config gpt2_1.5b_l8 --steps 1 > $O/rs.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_copy -s 60 -c 1 -o $O/copy -f \
    python scripts/sim_bench.py --ranks 4 --stage 3 --config gpt2_1.5b_l8 --steps 1 > $O/copy.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_mlp.csv \
    python bench.py --config mlp1m --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-fp16-key > $O/launches_mlp.log 2>&1
for r in adam flatten rs copy; do
  ncu -i $O/$r.ncu-rep --page raw --csv > $O/$r.raw.csv 2>/dev/null
  ncu -i $O/$r.ncu-rep --page details --csv > $O/$r.details.csv 2>/dev/null
done
# the .ncu-rep files are large: keep the CSV exports only (gpurun copies back <= 64 MiB)
mkdir -p /tmp/ncu_reps && mv $O/*.ncu-rep /tmp/ncu_reps/ 2>/dev/null
du -sh gpurun_out
