# full-size parity (config 2) and a config-3 bench
free -g | head -2; nproc
timeout 1800 python -m pytest tests -x -q -m "gpu and slow" 2>&1 | tail -5
BENCH_ALLOW_SHORT=1 timeout 900 python bench.py --config cfg3_sphere --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
python - <<'PY'
import json
try:
    d = json.loads(open('gpurun_out/bench_cfg3.json').read().strip().splitlines()[-1])
    print('cfg3 value %.3e ms %.3f iters %s' % (d['value'], d['ms_per_step'], d['config']['pcg_iters']))
    for k, v in d['kernels'].items(): print('  %-22s %8.3f ms  n=%4d  %s GB/s' % (k, v['ms_per_solve'], v['launches_per_solve'], v['gbs'] and round(v['gbs'])))
except Exception as e:
    print('cfg3 failed', e); print(open('gpurun_out/bench_cfg3.err').read()[-3000:])
PY
