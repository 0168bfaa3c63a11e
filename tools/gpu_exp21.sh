python tools/exp_build.py ry4d -DABFT_RY_F64=4 > /dev/null 2>&1
for l in base ry4d; do python tools/exp_modes.py $l cfg5 40 128 >> gpurun_out/exp21.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/t21.log 2>&1; tail -2 gpurun_out/t21.log
