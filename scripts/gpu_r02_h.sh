#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/prof
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
O=gpurun_out/prof
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_reduce_scatter -s 12 -c 1 -o $O/rs -f \
    python scripts/sim_bench.py --ranks 4 --stage 2 --config gpt2_1.5b_l8 --steps 1 > $O/rs.log 2>&1
ZERO_RS_MULTI=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_reduce_scatter -s 48 -c 1 -o $O/rs1 -f \
    python scripts/sim_bench.py --ranks 4 --stage 2 --config gpt2_1.5b_l8 --steps 1 > $O/rs1.log 2>&1
for r in rs rs1; do
  ncu -i $O/$r.ncu-rep --page raw --csv > $O/$r.raw.csv 2>/dev/null
  ncu -i $O/$r.ncu-rep --page details --csv > $O/$r.details.csv 2>/dev/null
done
mkdir -p /tmp/ncu_reps && mv $O/*.ncu-rep /tmp/ncu_reps/ 2>/dev/null
