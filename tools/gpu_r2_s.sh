#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/gputests.log
tail -2 gpurun_out/gputests.log; grep -E "^FAILED" gpurun_out/gputests.log | head -8
for cfg in cfg3_sphere cfg4_tank; do
  for v in "split:" "nosplit:OCTMG_PASS_SPLIT=0 OCTMG_RESTRICT_RED=0"; do
    tag=${v%%:*}; envs=${v#*:}
    env $envs timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-wcycle --no-cpu-baseline > gpurun_out/ab_${cfg}_${tag}.json 2> gpurun_out/ab_${cfg}_${tag}.err
    python -c "import json,sys; d=json.load(open('gpurun_out/ab_${cfg}_${tag}.json')); print('$cfg $tag', round(d['ms_per_step'],3), d['config']['pcg_iters'], {k:round(v['ms_per_solve'],3) for k,v in d['kernels'].items() if v['ms_per_solve']>0.5})" || tail -3 gpurun_out/ab_${cfg}_${tag}.err
  done
done
timeout 900 python tools/prof_levels.py cfg5_tank > gpurun_out/levels_cfg5_tank.txt 2>&1; head -12 gpurun_out/levels_cfg5_tank.txt
