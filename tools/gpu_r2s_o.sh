#!/bin/bash
# config-2 apply: ncu --set full with source, and the solve's launch list
mkdir -p gpurun_out/ncu2
export PATH=/usr/local/cuda/bin:$PATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
OCTMG_GRAPH_LOOP=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_apply_v6 -s 1 -c 1 -o gpurun_out/ncu2/apply \
      python tools/prof_solve.py cfg2_uniform256 0 > gpurun_out/ncu2/apply.log 2>&1
tail -1 gpurun_out/ncu2/apply.log
OCTMG_GRAPH_LOOP=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu2/launches_cfg2b.csv python tools/prof_solve.py cfg2_uniform256 2 > /dev/null 2>&1
ls -la gpurun_out/ncu2
