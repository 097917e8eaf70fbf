#!/bin/bash
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
rm -f gpurun_out/c3_*.ncu-rep
OCTMG_GRAPH_LOOP=0 timeout 600 ncu --set full --clock-control none --import-source on --warp-sampling-interval 2 -k regex:k_pass_v3 -s 2 -c 1 -o gpurun_out/c3_k_pass_v3 \
      python tools/prof_solve.py cfg3_sphere 0 > /dev/null 2>&1; echo "ncu rc=$?"
