# per-kernel durations (ncu, serialised) of the small-config launch sequence (tools/exp_small.py)
for c in cfg3 cfg2; do
  timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"k[123]_" --csv --log-file gpurun_out/small_$c.csv python tools/exp_small.py $c > /dev/null 2>&1; echo "$c rc=$?"
done
