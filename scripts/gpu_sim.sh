#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python scripts/sim_bench.py > gpurun_out/sim_bench.json 2> gpurun_out/sim_bench.err
timeout 600 python scripts/sim_bench.py --stage 1 > gpurun_out/sim_bench_s1.json 2>> gpurun_out/sim_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sim.csv \
    python scripts/sim_bench.py --steps 1 > gpurun_out/ncu_sim.log 2>&1
