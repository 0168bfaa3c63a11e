# GPU round (run through gpurun from the repo root): every GPU test, then the
# measurements of tools/gpu_final.sh (smoke, bench lines, reference arm, launch
# lists, ncu --set full of the top kernels -- each capture after its command
# ran clean without ncu)
timeout 2400 python -m pytest tests -m gpu -x -q -rs --durations=12 > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?
grep -E "FAILED|Error|passed|failed" gpurun_out/pytest.log | tail -8
bash tools/gpu_final.sh
