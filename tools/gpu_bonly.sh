# offline b-only (Q29): new GPU tests, IPC cases, offline suites; cfg5 bench line (lazy = b-only offline)
timeout 1500 python -m pytest tests/test_gpu_offline_bonly.py tests/test_ipc_multiprocess.py tests/test_gpu_parity.py -q -x -k "offline or bonly or lazy or partial" > gpurun_out/pytest_bonly.log 2>&1; echo pytest_rc=$?
grep -E "FAILED|Error|passed|failed" gpurun_out/pytest_bonly.log | tail -15
timeout 900 python bench.py --config cfg5 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo bench_rc=$?
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_cfg5.json").read().strip().splitlines()[-1])
r=d["roofline"]; o=d["other_policy"]
print("cfg5", d["value"], "ovh", d["abft_overhead_pct"], "ovh_flips", d["abft_overhead_with_flips_pct"], "both", o["abft_overhead_pct"], "prot", d["error_free_protected_gcells"], "unprot", d["unprotected_gcells"], "k1", r["k1_ms"], "k1u", r["k1_unprotected_ms"], "chk", r["check_ms_per_sweep"], "other k1", o["k1_ms"], "other chk", o["check_ms_per_sweep"], "clk", d["clocks"])
PY
tail -3 gpurun_out/bench_cfg5.err
