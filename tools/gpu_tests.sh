# GPU tests, then the bench with the fused check on / off (cfg4, cfg2, cfg3)
timeout 2400 python -m pytest tests -m gpu -x -q --durations=12 > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?
tail -25 gpurun_out/pytest.log
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e"
for cfg in cfg4 cfg2 cfg3; do
  for f in 1 0; do
    ABFT_FUSED_CHECK=$f timeout 600 $B --config $cfg > gpurun_out/bench_${cfg}_f$f.json 2> gpurun_out/bench_${cfg}_f$f.err
    python - <<PY
import json
d=json.loads(open("gpurun_out/bench_${cfg}_f$f.json").read().strip().splitlines()[-1])
r=d["roofline"]; o=d["other_policy"]
print("${cfg} fused=$f", d["value"], "ovh", d["abft_overhead_pct"], "ovh_flips", d["abft_overhead_with_flips_pct"], "both", o["abft_overhead_pct"], "k1", r["k1_ms"], "k1u", r["k1_unprotected_ms"], "chk", r["check_ms_per_sweep"], "clk", d["clocks"])
PY
  done
done
