# per-kernel durations (ncu, serialised) of NONE / LAZY serial / BOTH serial / LAZY pipelined step(20) on cfg2, cfg3
for c in cfg2 cfg3; do
  timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread --clock-control none --csv --log-file gpurun_out/small_$c.csv python tools/exp_small.py $c > gpurun_out/small_$c.log 2>&1
  echo "$c rc=$?"
done
