#!/bin/bash
# ZERO_RS_GRID: parity of capped pull grids, and the simulated N = 4 step vs the pull's grid
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/u
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_variants.py -q -k "rs_grid_cap" > $O/variants.log 2>&1; echo "rc=$?" >> $O/variants.log
tail -2 $O/variants.log
: > $O/rs_grid_sim.jsonl
for multi in 1 0; do
for g in 0 296 148 64 32 16; do
  r=$(ZERO_RS_MULTI=$multi ZERO_RS_GRID=$g timeout 600 python scripts/sim_bench.py --ranks 4 --stage 2 --config gpt2_1.5b --steps 10 2>>$O/err | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[1]); print(json.dumps({'rs_multi': $multi, 'rs_grid': $g, 'ms_per_step': d['ms_per_step'], 'effective_TBps': d['effective_TBps']}))" "$r" >> $O/rs_grid_sim.jsonl
done
done
cat $O/rs_grid_sim.jsonl
