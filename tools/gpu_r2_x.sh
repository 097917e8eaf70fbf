#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
for cfg in cfg2_uniform256 cfg3_sphere; do
  for v in "m16:" "m20:OCTMG_PASS_MINB=20"; do
    tag=${v%%:*}; envs=${v#*:}
    env $envs timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-wcycle --no-cpu-baseline > gpurun_out/ab_${cfg}_${tag}.json 2> gpurun_out/ab_${cfg}_${tag}.err
    python -c "import json,sys; d=json.load(open('gpurun_out/ab_${cfg}_${tag}.json')); print('$cfg $tag', round(d['ms_per_step'],3), d['config']['pcg_iters'], {k:round(v['ms_per_solve'],3) for k,v in d['kernels'].items() if k in ('residual_restrict','rbgs_pass','coarse_levels','prolong')})" || tail -3 gpurun_out/ab_${cfg}_${tag}.err
  done
done
