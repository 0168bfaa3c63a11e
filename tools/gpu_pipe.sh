# pipeline tests (pipelined / graphs / serial), then bench cfg4 new vs previous build
timeout 1200 python -m pytest tests/test_gpu_pipeline.py -q > gpurun_out/pytest_pipe.log 2>&1; echo pipe_rc=$?; grep -E "FAILED|passed|failed" gpurun_out/pytest_pipe.log | tail -25
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e"
for lib in new old; do
  if [ $lib = old ]; then export ABFT_LIB=$PWD/tools/explib/libabft_old.so; else unset ABFT_LIB; fi
  timeout 600 $B --config cfg4 > gpurun_out/bench_cfg4_$lib.json 2> gpurun_out/bench_cfg4_$lib.err
  python - <<PY
import json
d=json.loads(open("gpurun_out/bench_cfg4_$lib.json").read().strip().splitlines()[-1])
r=d["roofline"]; o=d["other_policy"]
print("cfg4 $lib", d["value"], "ovh", d["abft_overhead_pct"], "ovh_flips", d["abft_overhead_with_flips_pct"], "both", o["abft_overhead_pct"], "unprot", d["unprotected_gcells"], "k1", r["k1_ms"], "k1u", r["k1_unprotected_ms"], "chk", r["check_ms_per_sweep"], "clk", d["clocks"]["sm_mhz"], d["clocks"].get("reasons"))
PY
  tail -2 gpurun_out/bench_cfg4_$lib.err
done
