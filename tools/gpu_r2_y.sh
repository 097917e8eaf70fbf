#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/gputests.log
tail -2 gpurun_out/gputests.log; grep -E "^FAILED" gpurun_out/gputests.log | head -8
for cfg in cfg2_uniform256 cfg4_tank cfg5_tank; do
  for v in "warp:" "cta:OCTMG_WARP_COARSEST=0"; do
    tag=${v%%:*}; envs=${v#*:}
    env $envs timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-wcycle --no-cpu-baseline > gpurun_out/ab_${cfg}_${tag}.json 2> gpurun_out/ab_${cfg}_${tag}.err
    python -c "import json,sys; d=json.load(open('gpurun_out/ab_${cfg}_${tag}.json')); print('$cfg $tag', round(d['ms_per_step'],3), d['config']['pcg_iters'], {k:round(v['ms_per_solve'],3) for k,v in d['kernels'].items() if k in ('coarse_subcycle','coarse_levels')})" || tail -3 gpurun_out/ab_${cfg}_${tag}.err
  done
done
