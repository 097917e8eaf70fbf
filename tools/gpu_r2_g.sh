#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -m "gpu and not slow" -q -x > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/gputests.log
tail -2 gpurun_out/gputests.log; grep -E "^FAILED" gpurun_out/gputests.log | head -5
timeout 600 python tools/prof_levels.py cfg4_tank gpurun_out/levels_cfg4_tank.json > gpurun_out/levels_cfg4_tank.txt 2>&1; head -4 gpurun_out/levels_cfg4_tank.txt
OCTMG_GRAPH_LOOP=0 timeout 600 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:k_coarse_dense -s 6 -c 1 \
  -o gpurun_out/r02_coarse_dense python tools/prof_solve.py tank_mid 1 > gpurun_out/ncu_cd.log 2>&1; echo "ncu rc=$?"
