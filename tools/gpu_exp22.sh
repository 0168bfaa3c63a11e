python tools/exp_build.py ry8d -DABFT_RY_F64=8 > /dev/null 2>&1
for l in base ry8d; do python tools/exp_modes.py $l cfg5 40 128 >> gpurun_out/exp22.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/t22.log 2>&1; tail -2 gpurun_out/t22.log
