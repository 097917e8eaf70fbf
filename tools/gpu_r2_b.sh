#!/bin/bash
# build, fast GPU tests, cfg2 + cfg3 bench, cfg5 precision diagnostic
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/gputests.log
tail -3 gpurun_out/gputests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-wcycle --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench cfg2 rc=$?"
timeout 600 python bench.py --config cfg3_sphere --steps 10 --warmup 3 --no-wcycle --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "bench cfg3 rc=$?"
timeout 900 python tools/diag_cfg5.py > gpurun_out/diag5.log 2>&1; echo "diag rc=$?"
tail -6 gpurun_out/diag5.log
