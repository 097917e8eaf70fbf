# A/B of env-selected variants: bash tools/gpu_abenv.sh VAR "v1 v2 ..." [config]
VAR=$1; VALS=$2; CFG=${3:-cfg2_uniform256}
for V in $VALS; do
  echo "== $VAR=$V"
  env $VAR=$V python tools/time_vcycle.py $CFG 2>&1 | grep -vE "^ +\S+ +0.000"
done
