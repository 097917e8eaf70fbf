#!/bin/bash
# level-4 passes of config 2 in context (no cache flush): L2 hit rate, DRAM bytes, duration
mkdir -p gpurun_out/ncu2
export PATH=/usr/local/cuda/bin:$PATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
OCTMG_GRAPH_LOOP=0 timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:k_pass -s 40 -c 24 -o gpurun_out/ncu2/passes_ctx \
      python tools/prof_solve.py cfg2_uniform256 1 > gpurun_out/ncu2/passes_ctx.log 2>&1
tail -1 gpurun_out/ncu2/passes_ctx.log
OCTMG_GRAPH_LOOP=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu2/launches_cfg2.csv python tools/prof_solve.py cfg2_uniform256 2 > /dev/null 2>&1
ls -la gpurun_out/ncu2
