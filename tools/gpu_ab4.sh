OCTMG_SUBCYCLE_CTAS=8 timeout 1200 python -m pytest tests -x -q -m "gpu and not slow" -k "vcycle or pcg or schedule or loopback or mg" 2>&1 | tail -3
for C in cfg1_octant cfg2_uniform256 cfg4_tank; do
timeout 1500 python tools/ab_inproc.py $C '' 'OCTMG_SUBCYCLE_CTAS=8' 'OCTMG_SUBCYCLE_CTAS=8,OCTMG_SUBCYCLE_LD=2' 2>&1 | grep -E "==|subcycle"
done
