set -x
python tools/exp_build.py ry2b3 -DABFT_RY_F32=2 -DABFT_K1_MINB=3
python tools/exp_build.py ry2b4 -DABFT_RY_F32=2 -DABFT_K1_MINB=4
python tools/exp_build.py ry2b2 -DABFT_RY_F32=2 -DABFT_K1_MINB=2
for l in base ry2b3 ry2b4 ry2b2; do python tools/exp_modes.py $l >> gpurun_out/exp11.log 2>&1; done
cat gpurun_out/exp11.log
