#!/bin/bash
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest tests/test_gpu_sanitizer.py -q --durations=0 > gpurun_out/sanitizer.log 2>&1; echo "sanitizer rc=$?" >> gpurun_out/sanitizer.log
tail -15 gpurun_out/sanitizer.log
