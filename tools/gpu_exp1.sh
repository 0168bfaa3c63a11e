set -x
python tools/exp_modes.py base > gpurun_out/exp1.log 2>&1
python tools/exp_modes.py nok2 >> gpurun_out/exp1.log 2>&1
python tools/exp_modes.py nored >> gpurun_out/exp1.log 2>&1
python tools/exp_modes.py base >> gpurun_out/exp1.log 2>&1
cat gpurun_out/exp1.log
