#!/bin/bash
# k_reduce_scatter variants on N_d = 4 simulated ranks (GPT-2 1.5B block buckets, stage 2):
# per-launch device time from ncu (gpu__time_duration + DRAM bytes), one CSV per variant.
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/rs_sweep
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() {  # name, env...
  name=$1; shift
  env "$@" timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none -k regex:k_reduce_scatter --csv --log-file gpurun_out/rs_sweep/$name.csv \
      python scripts/sim_bench.py --ranks 4 --stage 2 --config gpt2_1.5b_l8 --steps 2 > gpurun_out/rs_sweep/$name.log 2>&1
}
run p_c6_u1 ZERO_RS_CTAS=6 ZERO_RS_U=1
run pipe_c4 ZERO_RS_CTAS=4 ZERO_RS_PIPE=1
run w16_c4 ZERO_RS_CTAS=4 ZERO_RS_PIPE=2
run w16_c6 ZERO_RS_CTAS=6 ZERO_RS_PIPE=2
run w16_c8 ZERO_RS_CTAS=8 ZERO_RS_PIPE=2
run w16p_c3 ZERO_RS_CTAS=3 ZERO_RS_PIPE=3
run w16p_c2 ZERO_RS_CTAS=2 ZERO_RS_PIPE=3
# the whole simulated step (no profiler), default variant
timeout 600 python scripts/sim_bench.py --ranks 4 --stage 2 > gpurun_out/rs_sweep/sim_step.jsonl 2>&1
