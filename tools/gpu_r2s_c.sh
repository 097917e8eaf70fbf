#!/bin/bash
# ncu --set full of the config-3 ghost-heavy kernels: apply, level-7 plain pass, ghost restriction
mkdir -p gpurun_out/ncu3
export PATH=/usr/local/cuda/bin:$PATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
for KS in k_apply_v6:0 k_pass_v3:2 k_restrict_row:0 k_inner_face_means:0; do
  K=${KS%%:*}; S=${KS##*:}
  OCTMG_GRAPH_LOOP=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/ncu3/$K \
      python tools/prof_solve.py cfg3_sphere 0 > gpurun_out/ncu3/$K.log 2>&1
  tail -2 gpurun_out/ncu3/$K.log
done
ls -la gpurun_out/ncu3
