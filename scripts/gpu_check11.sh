#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python scripts/train_bench.py --opt zero > gpurun_out/train_zero.json 2> gpurun_out/train_zero.err
timeout 900 python scripts/train_bench.py --opt torch > gpurun_out/train_torch.json 2> gpurun_out/train_torch.err
timeout 900 python scripts/train_bench.py --opt zero --stage 2 > gpurun_out/train_zero_s2.json 2> gpurun_out/train_zero_s2.err
