#!/bin/bash
# small-model latency work: GPU suite + config-1 eager/graph (L2 flushed per step and not)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/o
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
for pdl in 1 0; do
  for g in "" "--graph"; do
    ZERO_ADAM_PDL=$pdl timeout 120 python bench.py --config mlp1m $g --steps 400 --no-cpu-baseline --no-e2e --no-fp16-key > $O/mlp_pdl${pdl}${g}.json 2>> $O/mlp.err
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().splitlines()[-1]); print(sys.argv[1], round(d['ms_per_step']*1000,2), 'us', d['config']['l2'])" $O/mlp_pdl${pdl}${g}.json
  done
done
