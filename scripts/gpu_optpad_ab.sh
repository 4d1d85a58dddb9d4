#!/bin/bash
# DRAM channel balance: distance between the p32 / m / v arrays (ZERO_OPT_PAD elements)
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
: > gpurun_out/optpad.jsonl
for rep in 1 2; do
for pad in 0 1024 4160 65600 1048640; do
  ZERO_OPT_PAD=$pad timeout 600 python bench.py --config gpt2_1.5b --stage 1 --steps 50 --warmup 5 --no-e2e --no-fp16-key --no-cpu-baseline \
     | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'pad': $pad, 'ms': d['ms_per_step'], 'adam_ms': d['roofline']['ms_per_launch'], 'frac': d['roofline']['frac']}))" >> gpurun_out/optpad.jsonl
done
done
timeout 600 ncu --metrics dram__bytes.min.per_second,dram__bytes.max.per_second,dram__bytes.avg.per_second,gpu__time_duration.sum --clock-control none -k regex:k_adam -s 3 -c 1 --csv --log-file gpurun_out/optpad_ncu0.csv \
   python bench.py --config gpt2_1.5b --stage 1 --steps 1 --warmup 3 --no-e2e --no-fp16-key --no-cpu-baseline > /dev/null 2>&1
ZERO_OPT_PAD=4160 timeout 600 ncu --metrics dram__bytes.min.per_second,dram__bytes.max.per_second,dram__bytes.avg.per_second,gpu__time_duration.sum --clock-control none -k regex:k_adam -s 3 -c 1 --csv --log-file gpurun_out/optpad_ncu1.csv \
   python bench.py --config gpt2_1.5b --stage 1 --steps 1 --warmup 3 --no-e2e --no-fp16-key --no-cpu-baseline > /dev/null 2>&1
