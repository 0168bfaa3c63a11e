# GPU round: all GPU tests, smoke, bench lines (cfg4 headline + cfg5 slab),
# launch lists and ncu --set full captures (each after its command ran clean)
set -x
mkdir -p /tmp/nc
timeout 2400 python -m pytest tests -m gpu -x -q -rs --durations=12 > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?
tail -18 gpurun_out/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; tail -c 3000 gpurun_out/bench_cfg4.json
timeout 900 python bench.py --config cfg5 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; tail -c 2500 gpurun_out/bench_cfg5.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1; tail -c 800 gpurun_out/bench_ref.json
B4="python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv $B4 > gpurun_out/ncu_list4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_sweep -s 2 -c 1 -o /tmp/nc/k1_cfg4_lazy $B4 > gpurun_out/ncu_k1_4.log 2>&1
B5="python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv $B5 > gpurun_out/ncu_list5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_sweep -s 30 -c 1 -o /tmp/nc/k1_cfg5 $B5 > gpurun_out/ncu_k1_5.log 2>&1
for r in k1_cfg4_lazy k1_cfg5; do python tools/ncu_summary.py /tmp/nc/$r.ncu-rep > gpurun_out/$r.txt 2>&1; python tools/ncu_summary.py --sass /tmp/nc/$r.ncu-rep >> gpurun_out/$r.txt 2>&1; cp /tmp/nc/$r.ncu-rep gpurun_out/; done
ls -la gpurun_out
