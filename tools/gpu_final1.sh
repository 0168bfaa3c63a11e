timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/tests_final.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --config cfg5 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_cfg5.log 2>&1
timeout 300 python bench.py --config cfg3 --steps 200 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_cfg3.log 2>&1
timeout 300 python bench.py --config cfg2 --steps 100 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_cfg2.log 2>&1
timeout 900 python campaign.py --reps 100 --out gpurun_out/campaign.json > gpurun_out/campaign.log 2>&1
du -sh gpurun_out
