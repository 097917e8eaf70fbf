export PATH=/usr/local/cuda/bin:$PATH
K=${1:-k_smooth}
S=${2:-0}
C=${3:-2}
ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c $C -o gpurun_out/prof_$K python tools/prof_solve.py cfg2_uniform256 0 > gpurun_out/prof_$K.log 2>&1
tail -3 gpurun_out/prof_$K.log
