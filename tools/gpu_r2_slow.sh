#!/bin/bash
# build, then the full-size parity tests (-m "gpu and slow"); host facts recorded
mkdir -p gpurun_out
nproc > gpurun_out/slow_host.txt; free -g >> gpurun_out/slow_host.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
(while true; do date +%T | tr '\n' ' ' >> gpurun_out/slow_mem.log; free -g | sed -n 2p >> gpurun_out/slow_mem.log; sleep 60; done) &
MON=$!
timeout 3000 python -m pytest tests -m "gpu and slow" -q -s --durations=0 > gpurun_out/slowtests.log 2>&1; echo "slow tests rc=$?" >> gpurun_out/slowtests.log
kill $MON
tail -15 gpurun_out/slowtests.log
