#!/bin/bash
# k_reduce_scatter variants on simulated ranks (GPT-2 1.5B block buckets, stage 2): per-launch
# device time from ncu (gpu__time_duration + DRAM bytes), one CSV per (ranks, variant).
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/rs_sweep
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() {  # ranks, name, env...
  n=$1; name=$2; shift 2
  env "$@" timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none -k regex:k_reduce_scatter --csv --log-file gpurun_out/rs_sweep/n${n}_$name.csv \
      python scripts/sim_bench.py --ranks $n --stage 2 --config gpt2_1.5b_l8 --steps 2 > gpurun_out/rs_sweep/n${n}_$name.log 2>&1
}
for n in ${RS_RANKS:-2 4 8}; do
  run $n plain_u2_c4 ZERO_RS_PIPE=0 ZERO_RS_CTAS=4 ZERO_RS_U=2
  run $n plain_u1_c6 ZERO_RS_PIPE=0 ZERO_RS_CTAS=6 ZERO_RS_U=1
  run $n pipe_c4 ZERO_RS_CTAS=4 ZERO_RS_PIPE=1
  run $n pipe_c3 ZERO_RS_CTAS=3 ZERO_RS_PIPE=1
done
