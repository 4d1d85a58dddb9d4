#!/bin/bash
# config 1 A/B: flushed vs L2-resident, PDL on/off, eager/graph (interleaved, 2 rounds)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/p
mkdir -p $O
: > $O/mlp_ab.jsonl
for rep in 1 2; do
for fl in auto off; do
for pdl in 1 0; do
  for g in "" "--graph"; do
    r=$(ZERO_ADAM_PDL=$pdl timeout 120 python bench.py --config mlp1m $g --l2-flush $fl --steps 400 --no-cpu-baseline --no-e2e --no-fp16-key 2>>$O/err | tail -1)
    python - "$r" $fl $pdl "$g" >> $O/mlp_ab.jsonl <<'PY'
import json, sys
d = json.loads(sys.argv[1])
print(json.dumps({"l2_flush": sys.argv[2], "pdl": int(sys.argv[3]), "graph": bool(sys.argv[4]),
                  "us": d["ms_per_step"] * 1000, "p50_us": d["ms_per_step_p10_p50_p90"][1] * 1000}))
PY
  done
done
done
done
cat $O/mlp_ab.jsonl
