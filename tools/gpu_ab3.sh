timeout 1200 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | tail -4
timeout 900 python tools/ab_inproc.py cfg2_uniform256 '' 'OCTMG_SUBCYCLE_CTAS=1'
timeout 900 python tools/ab_inproc.py cfg1_octant '' 'OCTMG_SUBCYCLE_CTAS=1'
timeout 1500 python tools/ab_inproc.py cfg4_tank '' 'OCTMG_SUBCYCLE_CTAS=1'
