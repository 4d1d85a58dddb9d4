#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "ipc or checkpoint" > gpurun_out/pytest_sel.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sel.log
for st in 1 2 3; do
ZERO_BENCH_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2951$st \
   bench.py --gpus 2 --config gpt2_1.5b_l8 --stage $st --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_n2_s$st.json 2> gpurun_out/bench_n2_s$st.err
echo "rc=$?" >> gpurun_out/bench_n2_s$st.err
done
