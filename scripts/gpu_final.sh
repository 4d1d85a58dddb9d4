#!/bin/bash
# final round-2 validation on one B200: build, smoke, every GPU test, the contract bench line,
# the reference arm, the sanitizers
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
bash scripts/gpu_round.sh
bash scripts/sanitize.sh
