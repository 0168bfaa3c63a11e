for c in cfg2 cfg3; do timeout 600 python tools/exp_lib_ab.py $c base old 7 2>&1 | tail -2; done
timeout 900 python tools/exp_lib_ab.py cfg4 base old 5 2>&1 | tail -2
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv
timeout 1200 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_pipe.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest_pipe.log
