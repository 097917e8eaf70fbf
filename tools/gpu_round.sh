# Round check on one B200: smoke, GPU parity (not slow), default bench, launch list + ncu full of top kernels
export PATH=/usr/local/cuda/bin:$PATH
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader; nproc; free -g | head -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | tail -8
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python - <<'PY'
import json
try:
    d = json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
    print('value %.3e ms %.3f iters %s e2e %.3e' % (d['value'], d['ms_per_step'], d['config']['pcg_iters'], d['e2e']['value']))
    print('roofline', json.dumps(d['roofline']))
    for k, v in d['kernels'].items(): print('  %-22s %8.3f ms  n=%4d  %s GB/s' % (k, v['ms_per_solve'], v['launches_per_solve'], v['gbs'] and round(v['gbs'])))
    print('clocks', d['clocks'], 'launches', d['gpu_launches'], 'cpu', d.get('cpu_baseline'))
except Exception as e:
    print('bench parse failed', e); print(open('gpurun_out/bench.err').read()[-3000:])
PY
if [ "${PROFILES:-1}" = "1" ]; then bash tools/gpu_profiles.sh; fi
