#!/bin/bash
# build, fast GPU tests, bench (default + scalar-pass A/B), then the full-size parity tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/gputests.log
tail -3 gpurun_out/gputests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
OCTMG_PASS_V=2 timeout 300 python bench.py --steps 20 --warmup 5 --no-wcycle --no-cpu-baseline > gpurun_out/bench_v2.json 2> gpurun_out/bench_v2.err; echo "bench v2 rc=$?"
timeout 2400 python -m pytest tests -m "gpu and slow" -x -q -s > gpurun_out/slowtests.log 2>&1; echo "slow tests rc=$?" >> gpurun_out/slowtests.log
tail -3 gpurun_out/slowtests.log
