#!/bin/bash
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
rm -f gpurun_out/c3_*.ncu-rep
for KS in k_apply_v6:0 k_restrict_v2:0 k_pass_v3:2; do
  K=${KS%%:*}; S=${KS##*:}
  OCTMG_GRAPH_LOOP=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/c3_$K \
      python tools/prof_solve.py cfg3_sphere 0 > /dev/null 2>&1; echo "ncu $K rc=$?"
done
