#!/bin/bash
# build, fast GPU tests, per-level profiles of configs 2-5, ncu of the coarse sub-cycle and a
# small-level pass (tank_mid W-cycle: the same levels 0-2 as configs 4/5)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/gputests.log
tail -2 gpurun_out/gputests.log
for c in cfg2_uniform256 cfg3_sphere cfg4_tank cfg5_tank; do
  timeout 600 python tools/prof_levels.py $c gpurun_out/levels_$c.json > gpurun_out/levels_$c.txt 2>&1; cat gpurun_out/levels_$c.txt | head -20
done
OCTMG_GRAPH_LOOP=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_subcycle -s 6 -c 1 \
  -o gpurun_out/r02_subcycle python tools/prof_solve.py tank_mid 1 > gpurun_out/ncu_sub.log 2>&1; echo "ncu sub rc=$?"
OCTMG_GRAPH_LOOP=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pass_v2 -s 40 -c 1 \
  -o gpurun_out/r02_pass_small python tools/prof_solve.py tank_mid 1 > gpurun_out/ncu_pass.log 2>&1; echo "ncu pass rc=$?"
