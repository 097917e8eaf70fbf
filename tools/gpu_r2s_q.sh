#!/bin/bash
# fast GPU tests + A/B of an env-selected variant on configs 2 and 4 ($AB)
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?"
tail -2 gpurun_out/gputests.log; grep -E "^FAILED" gpurun_out/gputests.log | head -8
for C in ${CONFIGS:-cfg2_uniform256 cfg4_tank}; do
for E in "" $AB; do
  env $E timeout 600 python tools/prof_levels.py $C > gpurun_out/ab/${C}_$E.txt 2>&1
  echo "[$E] $(head -1 gpurun_out/ab/${C}_$E.txt)"; grep "level [345]:" gpurun_out/ab/${C}_$E.txt
done
done
