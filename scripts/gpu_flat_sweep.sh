#!/bin/bash
# flatten launch-shape sweep on one box: vectors in flight x CTAs/SM (3 streams), then streams
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for i in 1 2; do
  timeout 900 python scripts/sweep.py --adam "" --flat "${FLAT:-4x4,8x2,8x3,4x3,4x2,2x6,8x4}" > gpurun_out/flat_sweep_$i.jsonl 2>&1
  timeout 600 python scripts/sweep.py --adam "" --base "${SBASE:-ZERO_FLAT_VECS=8,ZERO_FLAT_CTAS=2}" --flat-streams "${STREAMS:-1,2,4}" > gpurun_out/flat_streams_$i.jsonl 2>&1
done
