# A/B: fused RB iterations vs per-colour passes; then GPU parity with the default
for V in fused_noshell split; do
  echo "== $V"
  OCTMG_RB=$V BENCH_ALLOW_SHORT=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$V.json 2> gpurun_out/bench_$V.err
  python - "$V" <<'PY'
import json, sys
try:
    d = json.loads(open('gpurun_out/bench_%s.json' % sys.argv[1]).read().strip().splitlines()[-1])
except Exception:
    print(open('gpurun_out/bench_%s.err' % sys.argv[1]).read()[-2000:]); raise SystemExit
print('value %.3e ms %.3f iters %s' % (d['value'], d['ms_per_step'], d['config']['pcg_iters']))
for k, v in d['kernels'].items(): print('  %-22s %8.3f ms  n=%4d  %s GB/s' % (k, v['ms_per_solve'], v['launches_per_solve'], v['gbs'] and round(v['gbs'])))
PY
done
timeout 900 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | tail -3
