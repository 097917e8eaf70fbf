#!/bin/bash
# build, fast GPU tests, per-level profiles of configs 2-5 (after a kernel change)
mkdir -p gpurun_out/levels
export PATH=/usr/local/cuda/bin:$PATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?"
tail -2 gpurun_out/gputests.log; grep -E "^FAILED|Error" gpurun_out/gputests.log | head -8
for C in ${CONFIGS:-cfg2_uniform256 cfg3_sphere cfg4_tank cfg5_tank}; do
  timeout 900 python tools/prof_levels.py $C gpurun_out/levels/$C.json > gpurun_out/levels/$C.txt 2>&1
  cat gpurun_out/levels/$C.txt
done
