# validate HEAD: all GPU tests, smoke, bench lines (cfg4 headline, small configs serial vs pipelined)
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=15 > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?
grep -E "FAILED|ERROR|passed|failed" gpurun_out/pytest.log | tail -30
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo bench_rc=$?; tail -c 3500 gpurun_out/bench_cfg4.json
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e"
for cfg in cfg2 cfg3; do for s in 0 1; do
  ABFT_SCHEDULE=$s timeout 600 $B --config $cfg > gpurun_out/bench_${cfg}_s$s.json 2> gpurun_out/bench_${cfg}_s$s.err
  python - <<PY
import json
d=json.loads(open("gpurun_out/bench_${cfg}_s$s.json").read().strip().splitlines()[-1])
r=d["roofline"]; o=d["other_policy"]
print("${cfg} sched=$s", d["value"], "ovh", d["abft_overhead_pct"], "ovh_flips", d["abft_overhead_with_flips_pct"], "both", o["abft_overhead_pct"], "k1", r["k1_ms"], "k1u", r["k1_unprotected_ms"], "chk", r["check_ms_per_sweep"], "clk", d["clocks"], d["config"].get("schedule"))
PY
done; done
