#!/bin/bash
# Every BASELINE config that fits one B200, through bench.py (N=1): the 7.5B layout (Fig. 1) at
# stages 1-3 and fp16 dynamic, GPT-2 1.5B at stages 0-3, the 1M-param MLP eager and as a CUDA
# graph; then the NEXT-1 training-step context (train_bench.py).
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
O=gpurun_out/configs.jsonl
: > $O
for st in 1 2 3; do
  timeout 900 python bench.py --config gpt_7.5b --stage $st --steps 20 --no-cpu-baseline --no-e2e --no-fp16-key >> $O 2>> gpurun_out/configs.err
done
for st in 0 1 2 3; do
  timeout 600 python bench.py --config gpt2_1.5b --stage $st --steps 50 --no-cpu-baseline --no-e2e --no-fp16-key >> $O 2>> gpurun_out/configs.err
done
timeout 600 python bench.py --config gpt2_1.5b --stage 1 --dtype fp16 --steps 50 --no-cpu-baseline --no-e2e >> $O 2>> gpurun_out/configs.err
timeout 600 python bench.py --config mlp1m --no-cpu-baseline --no-e2e --no-fp16-key >> $O 2>> gpurun_out/configs.err
timeout 600 python bench.py --config mlp1m --graph --no-cpu-baseline --no-e2e >> $O 2>> gpurun_out/configs.err
for opt in zero torch none; do
  timeout 900 python scripts/train_bench.py --opt $opt >> gpurun_out/train_bench.jsonl 2>> gpurun_out/train_bench.err
done
