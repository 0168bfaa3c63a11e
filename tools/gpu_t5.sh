set -x
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/tests5.log 2>&1; tail -3 gpurun_out/tests5.log
python tools/exp_modes.py base > gpurun_out/exp7.log 2>&1; cat gpurun_out/exp7.log
