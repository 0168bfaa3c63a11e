timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?
grep -E "FAILED|Error|passed|failed" gpurun_out/pytest.log | tail -8
bash tools/gpu_ab.sh
timeout 600 python tools/exp_offline.py cfg5 3 2>&1 | grep -v Warn
mkdir -p /tmp/nc
for lib in base old; do
  if [ $lib = old ]; then export ABFT_LIB=$PWD/tools/explib/libabft_old.so; else unset ABFT_LIB; fi
  timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum -k regex:k2_check --csv --log-file gpurun_out/k2_$lib.csv python tools/exp_small.py cfg3 > /dev/null 2>&1
  python tools/ncu_summary.py --launches gpurun_out/k2_$lib.csv | head -3
done
