set -x
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/tests3.log 2>&1; tail -5 gpurun_out/tests3.log
python tools/exp_modes.py base > gpurun_out/exp3.log 2>&1
ABFT_K1_MARCH=y python tools/exp_modes.py base >> gpurun_out/exp3.log 2>&1
ABFT_K1_MARCH=y ABFT_Y_PROMO256=1 python tools/exp_modes.py base >> gpurun_out/exp3.log 2>&1
python tools/exp_build.py nored2 -DABFT_EXP_NO_RED -DABFT_EXP_NO_K2 && python tools/exp_modes.py nored2 >> gpurun_out/exp3.log 2>&1
cat gpurun_out/exp3.log
