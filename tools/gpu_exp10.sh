set -x
python tools/exp_build.py rel5 -DABFT_K1_RELEASE=1 -DABFT_NS=5
python tools/exp_build.py rel4 -DABFT_K1_RELEASE=1 -DABFT_NS=4
python tools/exp_build.py ns5 -DABFT_NS=5
for l in base rel5 rel4 ns5; do python tools/exp_modes.py $l >> gpurun_out/exp10.log 2>&1; done
cat gpurun_out/exp10.log
