#!/bin/bash
# ncu --set full of config 3's adaptive-path kernels at HEAD: the apply (irregular body inlined),
# a level-7 colour pass (ghost body inlined), the ghost-tile residual-restriction
mkdir -p gpurun_out/ncu3b
export PATH=/usr/local/cuda/bin:$PATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
for KS in k_apply_v6:0 k_pass_v3:2 k_restrict_row:0; do
  K=${KS%%:*}; S=${KS##*:}
  OCTMG_GRAPH_LOOP=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/ncu3b/$K \
      python tools/prof_solve.py cfg3_sphere 0 > gpurun_out/ncu3b/$K.log 2>&1
  tail -1 gpurun_out/ncu3b/$K.log
done
