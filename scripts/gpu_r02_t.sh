#!/bin/bash
# launch list of the contract command on the final code (cold-cache, serialised: shares only)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/t
mkdir -p $O
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_7p5b.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-fp16-key > $O/launches_7p5b.log 2>&1
echo "rc=$?"
gzip -f $O/launches_7p5b.csv
ls -la $O
