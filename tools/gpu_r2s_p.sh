#!/bin/bash
# fast GPU tests + config-2 A/B of the ghost-free pass / lean apply instances
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?"
tail -2 gpurun_out/gputests.log; grep -E "^FAILED" gpurun_out/gputests.log | head -8
for r in 1 2; do
for E in "" OCTMG_RZ_FUSED=0; do
  env $E timeout 600 python tools/prof_levels.py cfg2_uniform256 > gpurun_out/ab/cfg2_$E.txt 2>&1
  echo "[$E] $(head -1 gpurun_out/ab/cfg2_$E.txt)"; grep "pcg vectors\|level 5" gpurun_out/ab/cfg2_$E.txt
done
done
