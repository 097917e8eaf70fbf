bash tools/gpu_quick.sh
for V in 600 5000; do
  echo "== OCTMG_GRID=1 OCTMG_GRID_TILES=$V"
  OCTMG_GRID=1 OCTMG_GRID_TILES=$V BENCH_ALLOW_SHORT=1 timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('value %.4e ms %.3f'%(d['value'], d['ms_per_step']))
for k,v in d['kernels'].items(): print('  %-22s %8.3f ms n=%4d'%(k, v['ms_per_solve'], v['launches_per_solve']))
" || tail -5 gpurun_out/ab.err
done
