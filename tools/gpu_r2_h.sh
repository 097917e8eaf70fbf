#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -m "gpu and not slow" -q -x > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/gputests.log
tail -2 gpurun_out/gputests.log; grep -E "^FAILED" gpurun_out/gputests.log | head -5
for t in 256 512 1024; do
  OCTMG_CD_THREADS=$t timeout 600 python tools/prof_levels.py cfg4_tank > gpurun_out/levels_cfg4_t$t.txt 2>&1; echo "threads $t"; head -3 gpurun_out/levels_cfg4_t$t.txt | sed -n '1p;3p'
done
