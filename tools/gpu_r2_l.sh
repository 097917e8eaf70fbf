#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -k "parity or variants" > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/gputests.log
tail -2 gpurun_out/gputests.log; grep -E "^FAILED" gpurun_out/gputests.log | head -8
for c in cfg2_uniform256 cfg4_tank cfg5_tank; do
  timeout 600 python tools/prof_levels.py $c gpurun_out/levels_$c.json > gpurun_out/levels_$c.txt 2>&1; head -5 gpurun_out/levels_$c.txt
done
