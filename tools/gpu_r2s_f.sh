#!/bin/bash
# ncu --set full of config 5's apply (inline irregular body) and level-9 pass
mkdir -p gpurun_out/ncu5
export PATH=/usr/local/cuda/bin:$PATH
for KS in k_apply_v6:0 k_pass_v3:2; do
  K=${KS%%:*}; S=${KS##*:}
  OCTMG_APPLY_IRR=inline OCTMG_GRAPH_LOOP=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/ncu5/$K \
      python tools/prof_solve_dev.py cfg5_tank 0 > gpurun_out/ncu5/$K.log 2>&1
  tail -1 gpurun_out/ncu5/$K.log
done
