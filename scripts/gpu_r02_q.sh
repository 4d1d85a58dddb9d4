#!/bin/bash
# DRAM traffic of the fused Adam at the contract config itself (7.5B, stage 2): a one-pass
# metric set under application replay (no 105 GB save/restore), plus the launch list
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/q
mkdir -p $O
timeout 1500 ncu --replay-mode application --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
   --clock-control none -k regex:k_adam -s 3 -c 1 --csv --log-file $O/adam_7p5b_dram.csv \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-fp16-key > $O/adam_7p5b.log 2>&1
echo "ncu rc=$?" >> $O/adam_7p5b.log
tail -5 $O/adam_7p5b.log
cat $O/adam_7p5b_dram.csv | tail -5
