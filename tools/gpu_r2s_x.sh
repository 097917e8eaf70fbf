#!/bin/bash
# ncu --set full (source) of one k_coarse_dense launch (levels 0-1) of config 4
mkdir -p gpurun_out/ncu4
export PATH=/usr/local/cuda/bin:$PATH
OCTMG_COARSE_CLUSTER=0 OCTMG_GRAPH_LOOP=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_coarse_dense -s 5 -c 1 -o gpurun_out/ncu4/dense \
      python tools/prof_solve_dev.py cfg4_tank 0 > gpurun_out/ncu4/dense.log 2>&1
tail -1 gpurun_out/ncu4/dense.log
