# offline speculation of the next window's first sweep: the offline suites, then per-window cost A/B
timeout 2400 python -m pytest tests -m gpu -x -q -k "offline or partial or bonly or cfg5 or persistent or window or cfg3" > gpurun_out/pytest_spec.log 2>&1; echo pytest_rc=$?
grep -E "FAILED|Error|passed|failed" gpurun_out/pytest_spec.log | tail -6
for v in 0 1; do echo "== ABFT_OFFLINE_SPEC=$v"; ABFT_OFFLINE_SPEC=$v timeout 600 python tools/exp_offline.py cfg3 5 2>&1 | grep -v Warn; done
