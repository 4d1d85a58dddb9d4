#!/bin/bash
# flatten launch shape at the 7.5B contract config: reduce phase (ms) per (streams, CTAs/SM)
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
: > gpurun_out/flat_ab.jsonl
for rep in 1 2; do
for spec in "3 4" "2 4" "4 4" "3 3" "3 6" "3 8"; do
  set -- $spec
  ZERO_FLAT_STREAMS=$1 ZERO_FLAT_CTAS=$2 timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-fp16-key --no-cpu-baseline \
     | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'streams': $1, 'ctas': $2, 'ms': d['ms_per_step'], 'reduce_ms': d['step_roofline']['reduce_phase_ms'], 'adam_ms': d['roofline']['ms_per_launch']}))" >> gpurun_out/flat_ab.jsonl
done
done
