#!/bin/bash
# robustness: the bit-exact parity suites under every non-default launch knob combination
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/env_matrix
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
T="tests/test_gpu_parity.py tests/test_gpu_stage_equivalence.py tests/test_gpu_edge.py tests/test_gpu_mp.py tests/test_gpu_graph.py tests/test_gpu_checkpoint.py tests/test_gpu_torch_zero.py"
run() { name=$1; shift; env "$@" timeout 900 python -m pytest $T -q -p no:cacheprovider > gpurun_out/env_matrix/$name.log 2>&1; echo "rc=$?" >> gpurun_out/env_matrix/$name.log; }
run round1_paths ZERO_SMALL_BUCKET=0 ZERO_ADAM_SMALL=0 ZERO_RS_PIPE=0 ZERO_RS_CTA_PARTIALS=0 ZERO_RS_U=2
run one_flat_stream ZERO_FLAT_STREAMS=1
run rs_per_rank ZERO_RS_MULTI=0
run flat_grid_combine ZERO_FLAT_CTA_PARTIALS=0
run adam_register_all ZERO_ADAM_VARIANT=0
