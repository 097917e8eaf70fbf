#!/bin/bash
# Round-2 evidence: fast + slow GPU suites, smoke, the default bench line (+ configs 1 and 3),
# the bench's launch list, ncu --set full of the config-2 hot kernels, per-level profiles
mkdir -p gpurun_out/levels
export PATH=/usr/local/cuda/bin:$PATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
nproc; free -g | head -2; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_r02.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['gpu_launches'], d['clocks'], {k:v['ms_per_solve'] for k,v in d.get('wcycle_configs',{}).items()})"
for C in cfg1_octant cfg3_sphere; do
  timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-wcycle > gpurun_out/bench_$C.json 2> gpurun_out/bench_$C.err
  python -c "import json; d=json.load(open('gpurun_out/bench_$C.json')); print('$C', d['value'], d['ms_per_step'], d['config'].get('pcg_iters'))" || tail -3 gpurun_out/bench_$C.err
done
OCTMG_GRAPH_LOOP=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-wcycle > gpurun_out/launches_bench_stdout.txt 2>&1; echo "launch list rc=$?"
for KS in k_pass_v3:2 k_apply_v6:0 k_restrict_red:0 k_prolong:2 k_update:0; do
  K=${KS%%:*}; S=${KS##*:}
  OCTMG_GRAPH_LOOP=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/full_$K \
      python tools/prof_solve.py cfg2_uniform256 0 > /dev/null 2>&1
done
ls gpurun_out/*.ncu-rep
for C in cfg2_uniform256 cfg3_sphere cfg4_tank cfg5_tank; do
  timeout 900 python tools/prof_levels.py $C gpurun_out/levels/$C.json > gpurun_out/levels/$C.txt 2>&1
  head -1 gpurun_out/levels/$C.txt
done
timeout 2400 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?"
tail -1 gpurun_out/gputests.log; grep -E "^FAILED" gpurun_out/gputests.log | head -8
timeout 3000 python -m pytest tests -m "gpu and slow" -q -s > gpurun_out/slowtests.log 2>&1; echo "slow tests rc=$?"
grep -E "cfg[0-9]|passed|failed" gpurun_out/slowtests.log | tail -8
