#!/bin/bash
# A/B: ghost value layers (new build) vs the in-place coarse gathers (ab/liboctmg_old.so), apply irregular body out of line vs inline
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out/ab
for C in cfg3_sphere cfg4_tank cfg5_tank; do
  for V in "new:" "new:OCTMG_APPLY_IRR=inline" "old:" "old:OCTMG_APPLY_IRR=inline"; do
    B=${V%%:*}; E=${V#*:}
    LIBV=""; [ "$B" = old ] && LIBV="OCTMG_LIB_AB=paper_2604_18886_b200/ab/liboctmg_old.so"
    env $LIBV $E timeout 600 python tools/prof_levels.py $C > gpurun_out/ab/${C}_${B}_${E}.txt 2>&1
    echo "[$B $E] $(head -1 gpurun_out/ab/${C}_${B}_${E}.txt)"; grep "pcg vectors" gpurun_out/ab/${C}_${B}_${E}.txt
  done
done
