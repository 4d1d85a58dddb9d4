#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python scripts/sweep.py --adam "" --flat 2x4,4x4,8x4,4x8,8x8,4x2 > gpurun_out/sweep5.jsonl 2> gpurun_out/sweep5.err
for st in 0 2 3; do timeout 300 python bench.py --stage $st --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/bench_stage$st.json 2>> gpurun_out/bench_stages.err; done
timeout 900 python bench.py --config gpt_7.5b --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_7p5b.json 2> gpurun_out/bench_7p5b.err
