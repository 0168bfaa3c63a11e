# closing checks of the round: GPU tests, smoke, bench (cfg4), campaign
mkdir -p gpurun_out/f3
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f3/tests.log 2>&1; tail -2 gpurun_out/f3/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/f3/bench.log 2>&1; echo bench rc=$?
timeout 900 python campaign.py --reps 100 --out gpurun_out/f3/campaign.json > gpurun_out/f3/campaign.log 2>&1; echo campaign rc=$?
