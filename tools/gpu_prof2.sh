# ncu --set full of named kernels inside one cfg2 solve: args "kernel:skip" ...
export PATH=/usr/local/cuda/bin:$PATH
for KS in "$@"; do
  K=${KS%%:*}; S=${KS##*:}
  ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/full_$K \
      python tools/prof_solve.py cfg2_uniform256 0 > gpurun_out/full_$K.log 2>&1
  tail -2 gpurun_out/full_$K.log
done
ls gpurun_out
