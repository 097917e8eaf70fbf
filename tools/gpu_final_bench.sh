export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print('cfg2', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'])" || tail -3 gpurun_out/bench.err
bash tools/gpu_profiles.sh > /dev/null 2>&1
for C in cfg1_octant cfg3_sphere cfg4_tank cfg5_tank; do
  timeout 1800 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$C.json 2> gpurun_out/bench_$C.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_$C.json').read().strip().splitlines()[-1]); print('$C', '%.4e'%d['value'], '%.2f ms'%d['ms_per_step'], d['config']['pcg_iters'])" || tail -3 gpurun_out/bench_$C.err
done
