#!/bin/bash
# round-2 validation after the config-1 latency change: build, smoke, GPU suite, the contract
# line + reference arm, config 1 (flushed / warm), its ncu launch list, the sanitizers
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${FINAL_DIR:-final2}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 300 python bench.py --config mlp1m --no-cpu-baseline --no-e2e --no-fp16-key > $O/mlp_eager.json 2> $O/mlp.err
timeout 300 python bench.py --config mlp1m --graph --no-cpu-baseline --no-e2e --no-fp16-key > $O/mlp_graph.json 2>> $O/mlp.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_mlp.csv \
    python bench.py --config mlp1m --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-fp16-key > $O/launches_mlp.log 2>&1
bash scripts/sanitize.sh > $O/sanitize.log 2>&1
cp -r gpurun_out/sanitize $O/ 2>/dev/null
tail -2 $O/pytest_gpu.log; tail -1 $O/smoke.log; grep -h 'rc=' $O/sanitize/*.log | sort | uniq -c
