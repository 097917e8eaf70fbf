#!/bin/bash
# GPU box: the config-5 oracle golden run (CPU, 12 threads) in the background, the fast GPU
# test suite + smoke in the foreground.
mkdir -p gpurun_out
(while true; do date +%T | tr '\n' ' ' >> gpurun_out/mem.log; free -g | sed -n 2p >> gpurun_out/mem.log; sleep 30; done) &
MON=$!
OMP_NUM_THREADS=12 python tools/oracle_golden_cfg5.py gpurun_out/cfg5_oracle.npz > gpurun_out/golden.log 2>&1 &
GP=$!
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
OMP_NUM_THREADS=4 timeout 2400 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gputests.log 2>&1
echo "gpu tests rc=$?" >> gpurun_out/gputests.log
OMP_NUM_THREADS=4 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
wait $GP
echo "golden rc=$?" >> gpurun_out/golden.log
kill $MON
