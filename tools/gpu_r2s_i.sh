#!/bin/bash
# build, the GMG tests, then the fast GPU suite
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_gmg.py -q -x > gpurun_out/gmg.log 2>&1; echo "gmg rc=$?"; tail -15 gpurun_out/gmg.log
timeout 1500 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?"
tail -2 gpurun_out/gputests.log; grep -E "^FAILED" gpurun_out/gputests.log | head -8
