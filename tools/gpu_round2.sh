set -x
timeout 1500 python -m pytest tests/test_ipc_multiprocess.py -x -q -rs > gpurun_out/pytest_ipc.log 2>&1; echo ipc_rc=$?
tail -30 gpurun_out/pytest_ipc.log
timeout 2400 python -m pytest tests -m gpu -x -q -rs --durations=12 --ignore=tests/test_ipc_multiprocess.py > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?
tail -22 gpurun_out/pytest.log
B4="python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv $B4 > gpurun_out/ncu_list4.log 2>&1
ls -la gpurun_out
