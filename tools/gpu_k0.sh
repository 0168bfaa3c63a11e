# all GPU tests (K0 feeds every parity case), then the cfg4 / cfg5 K0 launch times
timeout 2400 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?
grep -E "FAILED|Error|passed|failed" gpurun_out/pytest.log | tail -15
B4="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k0_ --csv --log-file gpurun_out/k0_cfg4.csv $B4 > /dev/null 2>&1; echo ncu4_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k0_ --csv --log-file gpurun_out/k0_cfg5.csv $B4 --config cfg5 > /dev/null 2>&1; echo ncu5_rc=$?
python tools/ncu_summary.py --launches gpurun_out/k0_cfg4.csv | head -8
python tools/ncu_summary.py --launches gpurun_out/k0_cfg5.csv | head -8
