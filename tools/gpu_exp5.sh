set -x
python tools/exp_build.py nocol -DABFT_EXP_NO_K2 -DABFT_EXP_NO_COLSUM
python tools/exp_build.py nored -DABFT_EXP_NO_K2 -DABFT_EXP_NO_RED
python tools/exp_build.py nok2 -DABFT_EXP_NO_K2
python tools/exp_build.py ry2 -DABFT_EXP_NO_K2 -DABFT_RY_F32=2
for l in base nok2 nocol nored ry2; do python tools/exp_modes.py $l >> gpurun_out/exp5.log 2>&1; done
cat gpurun_out/exp5.log
