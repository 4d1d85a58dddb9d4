#!/bin/bash
# the N > 1 bench flow on the final code (ranks share one GPU: functional), incl. the L2-flushed
# small config at N = 2, and the driver-style torchrun launch at N = 2
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r
mkdir -p $O
ZERO_BENCH_SAME_DEVICE=1 timeout 600 python bench.py --gpus 2 --stage 2 --config gpt2_1.5b_l8 --steps 3 --warmup 3 --no-cpu-baseline > $O/n2_l8.json 2> $O/n2_l8.err; echo "rc=$?" >> $O/n2_l8.err
ZERO_BENCH_SAME_DEVICE=1 timeout 600 python bench.py --gpus 2 --stage 2 --config mlp1m --steps 20 --warmup 3 --no-cpu-baseline --no-fp16-key > $O/n2_mlp.json 2> $O/n2_mlp.err; echo "rc=$?" >> $O/n2_mlp.err
ZERO_BENCH_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 \
   bench.py --gpus 2 --stage 3 --config gpt2_1.5b_l8 --steps 3 --warmup 3 --no-cpu-baseline > $O/n2_tr_s3.json 2> $O/n2_tr_s3.err; echo "rc=$?" >> $O/n2_tr_s3.err
for f in n2_l8 n2_mlp n2_tr_s3; do
  tail -1 $O/$f.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['n_gpus'], d['config']['workload'], round(d['ms_per_step'],3), d['comm']['equal'], d['config']['l2'][:40], d.get('e2e',{}).get('value'))" $O/$f.json
done
