#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in mlp1m gpt2_1.5b; do
  timeout 600 python bench.py --config $c --graph --no-cpu-baseline --no-e2e > gpurun_out/bench_graph_$c.json 2> gpurun_out/bench_graph_$c.err
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/bench_eager_$c.json 2> gpurun_out/bench_eager_$c.err
done
