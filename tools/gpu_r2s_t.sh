#!/bin/bash
# ncu --set full (source) of one k_coarse_cluster launch of config 4 (W-cycle)
mkdir -p gpurun_out/ncu4
export PATH=/usr/local/cuda/bin:$PATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
OCTMG_GRAPH_LOOP=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_coarse_cluster -s 5 -c 1 -o gpurun_out/ncu4/cluster \
      python tools/prof_solve_dev.py cfg4_tank 0 > gpurun_out/ncu4/cluster.log 2>&1
tail -1 gpurun_out/ncu4/cluster.log
