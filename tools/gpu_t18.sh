timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/t18.log 2>&1; tail -2 gpurun_out/t18.log
for l in base base; do python tools/exp_modes.py $l >> gpurun_out/exp18.log 2>&1; done
timeout 600 python campaign.py --exp e1 --reps 30 --out gpurun_out/c_e1b.json > /dev/null 2>&1
