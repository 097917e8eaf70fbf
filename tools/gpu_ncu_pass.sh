export PATH=/usr/local/cuda/bin:$PATH
ncu --set full --clock-control none --import-source on -k regex:k_pass_v2 -s 2 -c 1 -o gpurun_out/split_pass python tools/prof_solve.py cfg2_uniform256 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_apply -s 1 -c 1 -o gpurun_out/split_apply python tools/prof_solve.py cfg2_uniform256 0 > /dev/null 2>&1
ls gpurun_out/split_*
