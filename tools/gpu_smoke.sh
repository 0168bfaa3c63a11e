timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --config cfg2 --steps 100 --warmup 5 --no-cpu > gpurun_out/bench_cfg2.log 2>&1
timeout 900 python bench.py --config cfg3 --steps 200 --warmup 5 --no-cpu > gpurun_out/bench_cfg3.log 2>&1
