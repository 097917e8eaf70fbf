#!/bin/bash
# build, fast GPU tests, A/B of the ghost-body placement on configs 2/3/4, then the slow tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/gputests.log
tail -3 gpurun_out/gputests.log
for cfg in cfg2_uniform256 cfg3_sphere cfg4_tank; do
  for v in "base:" "passinl:OCTMG_PASS_GHOST=inline" "applyinl:OCTMG_APPLY_IRR=inline" "both:OCTMG_PASS_GHOST=inline OCTMG_APPLY_IRR=inline"; do
    tag=${v%%:*}; envs=${v#*:}
    if [ $cfg = cfg2_uniform256 ] && [ $tag != base ]; then continue; fi
    env $envs timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-wcycle --no-cpu-baseline > gpurun_out/ab_${cfg}_${tag}.json 2> gpurun_out/ab_${cfg}_${tag}.err
    python -c "import json,sys; d=json.load(open('gpurun_out/ab_${cfg}_${tag}.json')); print('$cfg $tag', round(d['ms_per_step'],3), d['config']['pcg_iters'], {k:round(v['ms_per_solve'],3) for k,v in d['kernels'].items() if v['ms_per_solve']>0.3})" || tail -3 gpurun_out/ab_${cfg}_${tag}.err
  done
done
timeout 3000 python -m pytest tests -m "gpu and slow" -q -s > gpurun_out/slowtests.log 2>&1; echo "slow tests rc=$?" >> gpurun_out/slowtests.log
grep -E "cfg[0-9]|passed|failed" gpurun_out/slowtests.log | tail -8
