# A/B of env-selected variants on the short bench: bash tools/gpu_abbench.sh VAR "v1 v2 ..." [config]
VAR=$1; VALS=$2; CFG=${3:-cfg2_uniform256}
for V in $VALS; do
  env $VAR=$V BENCH_ALLOW_SHORT=1 timeout 600 python bench.py --config $CFG --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$V.json 2> gpurun_out/ab_$V.err
  python - "$V" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f'gpurun_out/ab_{v}.json').read().strip().splitlines()[-1])
    print('== %s  value %.4e  ms %.3f  iters %s' % (v, d['value'], d['ms_per_step'], d['config']['pcg_iters']))
    for k, x in d['kernels'].items(): print('  %-22s %8.3f ms  n=%4d  %s GB/s' % (k, x['ms_per_solve'], x['launches_per_solve'], x['gbs'] and round(x['gbs'])))
except Exception as e:
    print('parse failed', v, e); print(open(f'gpurun_out/ab_{v}.err').read()[-2000:])
PY
done
