# Round profiles: launch list of the bench command + ncu --set full of the top kernels
# (launch list with the host-driven PCG loop: ncu does not list the kernels inside the
# conditional-while body of the device-side loop; the kernels are the same)
export PATH=/usr/local/cuda/bin:$PATH
if [ "${SKIP_LAUNCHES:-0}" != "1" ]; then
OCTMG_GRAPH_LOOP=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/launches_bench_stdout.txt 2>&1
fi
# launch indices inside one solve of config 2: level-5 plain pass = 3rd k_pass_v2 launch,
# level-5 prolongation = 4th k_prolong launch, the rest: first launch
for KS in k_pass_v2:2 k_apply:0 k_restrict:0 k_prolong:3 k_update:0; do
  K=${KS%%:*}; S=${KS##*:}
  OCTMG_GRAPH_LOOP=0 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/full_$K \
      python tools/prof_solve.py cfg2_uniform256 0 > /dev/null 2>&1
done
ls gpurun_out | tail -12
