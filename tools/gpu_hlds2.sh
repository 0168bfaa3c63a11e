timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?
grep -E "FAILED|Error|passed|failed" gpurun_out/pytest.log | tail -5
timeout 900 python bench.py --config cfg5 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo b5=$?
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_cfg5.json").read().strip().splitlines()[-1])
r=d["roofline"]; o=d["other_policy"]
print("cfg5", d["value"], "ovh", d["abft_overhead_pct"], "other", o["abft_overhead_pct"], "prot", d["error_free_protected_gcells"], "unprot", d["unprotected_gcells"], "k1", r["k1_ms"], "k1u", r["k1_unprotected_ms"], "frac", r["frac"], d["clocks"])
PY
