timeout 1200 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_gpu_geometry.py -x -q -m "gpu and slow" 2>&1 | tail -3
for C in cfg4_tank cfg5_tank; do
  timeout 1800 python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$C.json 2> gpurun_out/bench_$C.err
  python - "$C" <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.loads(open(f'gpurun_out/bench_{c}.json').read().strip().splitlines()[-1])
    print('%s value %.4e ms %.3f iters %s leaves %d e2e %.3e' % (c, d['value'], d['ms_per_step'], d['config']['pcg_iters'], d['config']['leaf_cells'], d['e2e']['value']))
    for k, v in d['kernels'].items(): print('  %-22s %8.3f ms  n=%4d  %s GB/s' % (k, v['ms_per_solve'], v['launches_per_solve'], v['gbs'] and round(v['gbs'])))
except Exception as e:
    print(c, 'failed', e); print(open(f'gpurun_out/bench_{c}.err').read()[-2000:])
PY
done
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
