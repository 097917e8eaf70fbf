#!/bin/bash
# re-entry check of HEAD: build, smoke, fast GPU tests, default bench
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
nproc; free -g | head -2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/gputests.log
tail -2 gpurun_out/gputests.log; grep -E "^FAILED" gpurun_out/gputests.log | head -8
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print('cfg2', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d.get('extra'))" || tail -3 gpurun_out/bench.err
