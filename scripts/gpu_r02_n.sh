#!/bin/bash
# config 1 launch-shape sensitivity (eager and graph)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/mlp_sweep.jsonl
: > $O
run() {  # env... -- label
  for g in "" "--graph"; do
    r=$(env "$@" timeout 120 python bench.py --config mlp1m $g --steps 400 --no-cpu-baseline --no-e2e --no-fp16-key 2>/dev/null | tail -1)
    python - "$r" "$*" "$g" >> $O <<'PY'
import json, sys
try: d = json.loads(sys.argv[1]); us = d["ms_per_step"] * 1000
except Exception: us = None
print(json.dumps({"env": sys.argv[2], "graph": bool(sys.argv[3]), "us": us}))
PY
  done
}
run X=0
run ZERO_FLAT_CTAS=1
run ZERO_FLAT_CTAS=2
run ZERO_FLAT_CTAS=8
run ZERO_FLAT_VECS=1
run ZERO_FLAT_CTAS=1 ZERO_FLAT_VECS=1
run ZERO_ADAM_PDL=0
run ZERO_STEP_SMALL=1
run ZERO_STEP_SMALL=1 ZERO_STEP_SMALL_CTAS=148
run ZERO_STEP_SMALL=1 ZERO_STEP_SMALL_CTAS=296
run ZERO_FLAT_CTA_PARTIALS=0
run ZERO_SMALL_BUCKET=0
cat $O
