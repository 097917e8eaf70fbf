set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; free -g | head -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 900 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt | tail -30
BENCH_ALLOW_SHORT=1 timeout 600 python bench.py --steps 3 --warmup 3 --cpu-seconds 5 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
tail -c 3000 gpurun_out/bench1.json; tail -20 gpurun_out/bench1.err
