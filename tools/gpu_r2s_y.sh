#!/bin/bash
# the level-3 cluster: its parity tests first, then the fast suite and configs 2/4/5
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out/levels
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -k "cluster_level3" -q -x > gpurun_out/c3.log 2>&1; echo "c3 rc=$?"; tail -15 gpurun_out/c3.log
timeout 900 python tools/prof_levels.py cfg2_uniform256 > gpurun_out/levels/c3_cfg2.txt 2>&1; head -5 gpurun_out/levels/c3_cfg2.txt
