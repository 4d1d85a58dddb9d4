#!/bin/bash
# flatten epilogue without the last-CTA combine (default) and PDL-chained flattens on one stream
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
ZERO_FLAT_PDL=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py tests/test_gpu_graph.py -m gpu -q -x > gpurun_out/pytest_pdl.log 2>&1; echo rc=$? >> gpurun_out/pytest_pdl.log
for i in 1 2 3; do
  timeout 900 python scripts/sweep.py --adam "" --env "ZERO_FLAT_PDL=0|ZERO_FLAT_PDL=1|ZERO_FLAT_PDL=0,ZERO_FLAT_STREAMS=4" > gpurun_out/pdl_sweep_$i.jsonl 2>&1
done
