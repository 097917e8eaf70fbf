for V in halo direct; do
  echo "== $V"
  OCTMG_TILE=$V python tools/time_vcycle.py 2>&1 | grep -E "rbgs|restrict|total|coarse"
done
OCTMG_TILE=halo timeout 900 python -m pytest tests -x -q -m "gpu and not slow" -k "vcycle or pcg" 2>&1 | tail -3
