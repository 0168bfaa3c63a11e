timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/t16.log 2>&1; tail -2 gpurun_out/t16.log
python tools/exp_modes.py base > gpurun_out/exp16.log 2>&1
python tools/exp_modes.py base >> gpurun_out/exp16.log 2>&1
