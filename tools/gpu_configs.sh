# BASELINE configs 3 and 4 on one B200 (bench lines), NCCL 2-rank check, round profiles, full-size parity
export PATH=/usr/local/cuda/bin:$PATH
# (NCCL refuses two ranks on one GPU: "invalid usage"; the NCCL path needs >= 2 GPUs)
for C in cfg1_octant cfg3_sphere cfg4_tank; do
  timeout 1500 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$C.json 2> gpurun_out/bench_$C.err
  tail -1 gpurun_out/bench_$C.err
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
[ "${PROFILES:-0}" = "1" ] && bash tools/gpu_profiles.sh
timeout 1200 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | tail -4
