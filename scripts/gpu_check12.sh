#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python scripts/sweep.py --adam "" --flat-streams 1,2,3,4 > gpurun_out/sweep7.jsonl 2> gpurun_out/sweep7.err
timeout 1200 python scripts/sweep.py --adam "" --flat 4x2,4x3,8x2,2x2 --base ZERO_FLAT_STREAMS=3 > gpurun_out/sweep8.jsonl 2> gpurun_out/sweep8.err
