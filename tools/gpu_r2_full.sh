#!/bin/bash
# the whole GPU suite (fast + slow), smoke, and the default bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/gputests.log
tail -2 gpurun_out/gputests.log; grep -E "^FAILED" gpurun_out/gputests.log | head -8
timeout 3000 python -m pytest tests -m "gpu and slow" -q -s > gpurun_out/slowtests.log 2>&1; echo "slow tests rc=$?" >> gpurun_out/slowtests.log
grep -E "cfg[0-9]|passed|failed" gpurun_out/slowtests.log | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_r02.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['gpu_launches'], {k:v['ms_per_solve'] for k,v in d['wcycle_configs'].items()})"
