# GPU round: tests, bench lines (cfg4 headline + cfg5 slab), launch lists and
# one ncu --set full capture of the cfg5 K1 (after the same command ran clean)
set -x
timeout 2400 python -m pytest tests -m gpu -x -q -rs --durations=12 > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?
tail -22 gpurun_out/pytest.log
timeout 900 python bench.py --config cfg5 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; tail -c 2500 gpurun_out/bench_cfg5.json
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; tail -c 2500 gpurun_out/bench_cfg4.json
B="python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu --no-e2e"
timeout 600 $B > gpurun_out/plain_cfg5.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv $B > gpurun_out/ncu_list.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_sweep -s 30 -c 1 -o gpurun_out/k1_cfg5 $B > gpurun_out/ncu_k1.log 2>&1
B4="python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv $B4 > gpurun_out/ncu_list4.log 2>&1
ls -la gpurun_out
