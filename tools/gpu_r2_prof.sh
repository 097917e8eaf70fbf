#!/bin/bash
# Round-2 evidence: default bench line, launch list of the bench command (host-driven loop so
# ncu lists the loop body), ncu --set full of the top kernels of config 2 (level 5 / leaves),
# and of the dense coarse cycle (tank_mid)
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; echo "bench rc=$?"
OCTMG_GRAPH_LOOP=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-wcycle > gpurun_out/launches_bench_stdout.txt 2>&1; echo "launches rc=$?"
rm -f gpurun_out/full_*.ncu-rep
for KS in k_pass_v3:2 k_apply_v6:0 k_restrict_red:0 k_prolong:3 k_update:0 k_dot_rz:0 k_coarse_cluster:0; do
  K=${KS%%:*}; S=${KS##*:}
  OCTMG_GRAPH_LOOP=0 timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/full_$K \
      python tools/prof_solve.py cfg2_uniform256 0 > /dev/null 2>&1; echo "ncu $K rc=$?"
done
