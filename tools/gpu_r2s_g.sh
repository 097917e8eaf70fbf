#!/bin/bash
# A/B of the apply's irregular-body placement / occupancy (OCTMG_APPLY_IRR)
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
for C in ${CONFIGS:-cfg3_sphere cfg5_tank cfg2_uniform256}; do
  for E in ${VARIANTS:-"" OCTMG_APPLY_IRR=inline7 OCTMG_APPLY_IRR=inline8 OCTMG_APPLY_IRR=call}; do
    env $E timeout 600 python tools/prof_levels.py $C > gpurun_out/ab/${C}_$E.txt 2>&1
    echo "[$E] $(head -1 gpurun_out/ab/${C}_$E.txt)"; grep "pcg vectors" gpurun_out/ab/${C}_$E.txt
  done
done
