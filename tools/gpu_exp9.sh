set -x
python tools/exp_build.py ku8 -DABFT_KU=8
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/t9.log 2>&1; tail -2 gpurun_out/t9.log
python tools/exp_modes.py base > gpurun_out/exp9.log 2>&1
python tools/exp_modes.py ku8 >> gpurun_out/exp9.log 2>&1
python tools/exp_modes.py base >> gpurun_out/exp9.log 2>&1
cat gpurun_out/exp9.log
