set -x
python tools/exp_build.py nok2 -DABFT_EXP_NO_K2
python tools/exp_build.py nocol -DABFT_EXP_NO_K2 -DABFT_EXP_NO_COLSUM
python tools/exp_build.py w4 -DABFT_EXP_NO_K2 -DABFT_WARPS=4
python tools/exp_build.py w4nocol -DABFT_EXP_NO_K2 -DABFT_WARPS=4 -DABFT_EXP_NO_COLSUM
python tools/exp_build.py ns4 -DABFT_EXP_NO_K2 -DABFT_NS=4
for l in nok2 nocol w4 w4nocol ns4; do python tools/exp_modes.py $l >> gpurun_out/exp4.log 2>&1; done
cat gpurun_out/exp4.log
