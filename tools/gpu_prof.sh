set -x
export PATH=/usr/local/cuda/bin:$PATH
# launch list of one profiled solve (warm-up solve skipped by launch count in post-processing)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python tools/prof_solve.py cfg2_uniform256 1 > gpurun_out/launches_stdout.txt 2>&1
# full sets of the dominant kernels
ncu --set full --clock-control none --import-source on -k regex:k_pass -s 1 -c 2 -o gpurun_out/prof_pass python tools/prof_solve.py cfg2_uniform256 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_apply -s 0 -c 1 -o gpurun_out/prof_apply python tools/prof_solve.py cfg2_uniform256 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_restrict -s 0 -c 1 -o gpurun_out/prof_restrict python tools/prof_solve.py cfg2_uniform256 0 > /dev/null 2>&1
ls -la gpurun_out
