# quick GPU check: smoke, GPU parity tests (not slow), short bench with per-kernel table
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | tail -6
BENCH_ALLOW_SHORT=1 timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
python - <<'PY'
import json
try:
    d = json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
    print('value %.4e ms %.3f iters %s e2e %.3e' % (d['value'], d['ms_per_step'], d['config']['pcg_iters'], d['e2e']['value']))
    print('roofline', json.dumps(d['roofline']))
    for k, v in d['kernels'].items(): print('  %-22s %8.3f ms  n=%4d  %s GB/s' % (k, v['ms_per_solve'], v['launches_per_solve'], v['gbs'] and round(v['gbs'])))
except Exception as e:
    print('bench parse failed', e); print(open('gpurun_out/bench.err').read()[-3000:])
PY
