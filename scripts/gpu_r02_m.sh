#!/bin/bash
# config 1 (1M-param MLP, stage 2, N = 1): where the 2-kernel step's ~21 us go
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/mlp_prof
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python bench.py --config mlp1m --no-cpu-baseline --no-e2e --no-fp16-key > $O/eager.json 2> $O/eager.err
timeout 300 python bench.py --config mlp1m --graph --no-cpu-baseline --no-e2e --no-fp16-key > $O/graph.json 2>> $O/eager.err
for cc in none all; do
  timeout 600 ncu --set full --clock-control none --cache-control $cc --import-source on -k regex:'k_flatten|k_adam' -s 20 -c 2 -o $O/mlp_$cc -f \
    python bench.py --config mlp1m --steps 3 --warmup 10 --no-e2e --no-cpu-baseline --no-fp16-key > $O/ncu_$cc.log 2>&1
  ncu -i $O/mlp_$cc.ncu-rep --page raw --csv > $O/mlp_$cc.raw.csv 2>/dev/null
  ncu -i $O/mlp_$cc.ncu-rep --page details --csv > $O/mlp_$cc.details.csv 2>/dev/null
  ncu -i $O/mlp_$cc.ncu-rep --page source --csv --print-source sass > $O/mlp_$cc.source.csv 2>/dev/null
done
rm -f $O/*.ncu-rep
du -sh $O
