# schedule A/B (tools/exp_sched.py) on cfg2 / cfg3 / cfg4
for c in cfg2 cfg3; do timeout 600 python tools/exp_sched.py $c 7 20 2>&1 | tail -12; done
timeout 900 python tools/exp_sched.py cfg4 3 20 2>&1 | tail -12
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv
