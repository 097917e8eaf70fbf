export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | tail -3
timeout 900 python tools/ab_inproc.py cfg1_octant '' 'OCTMG_SUBCYCLE_CTAS=8' 2>&1 | grep "=="
ncu --set full --clock-control none --import-source on -k regex:k_subcycle -s 2 -c 1 -o gpurun_out/sub_cfg1 python tools/prof_solve.py cfg1_octant 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pass_v2 -s 40 -c 1 -o gpurun_out/pass_l3 python tools/prof_solve.py uniform128 0 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
