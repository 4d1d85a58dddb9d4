#!/bin/bash
# flatten body at the 7.5B contract config: vectors in flight per thread and the TMA variants
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/s
mkdir -p $O
: > $O/flat_body_ab.jsonl
for rep in 1 2; do
for spec in "ZERO_FLAT_VECS=4" "ZERO_FLAT_VECS=2" "ZERO_FLAT_VECS=1" "ZERO_FLAT_TMA=1" "ZERO_FLAT_TMA=2"; do
  env $spec timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-fp16-key --no-cpu-baseline 2>>$O/err \
     | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'knob': '$spec', 'ms': d['ms_per_step'], 'reduce_ms': d['step_roofline']['reduce_phase_ms'], 'flatten_gbs': d['step_roofline']['flatten_gbs'], 'adam_ms': d['roofline']['ms_per_launch']}))" >> $O/flat_body_ab.jsonl
done
done
cat $O/flat_body_ab.jsonl
