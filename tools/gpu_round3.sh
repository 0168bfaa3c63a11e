set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg5 or box27 or partial or persistent" > gpurun_out/pytest_box.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest_box.log
timeout 900 python bench.py --config cfg5 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; tail -c 1500 gpurun_out/bench_cfg5.json
B="python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_sweep -s 30 -c 1 -o gpurun_out/k1_cfg5 $B > gpurun_out/ncu_k1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_sweepIdLi3ELi1 -c 1 -o gpurun_out/k1_cfg5_ab $B > gpurun_out/ncu_k1ab.log 2>&1
timeout 2400 python campaign.py --exp e1,e3 --reps 20 --out gpurun_out/campaign.json > gpurun_out/campaign.log 2>&1; echo camp=$?
ls -la gpurun_out
