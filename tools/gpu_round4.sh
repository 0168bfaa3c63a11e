set -x
timeout 1500 python -m pytest tests/test_ipc_multiprocess.py -x -q -rs > gpurun_out/pytest_ipc.log 2>&1; echo ipc_rc=$?
tail -5 gpurun_out/pytest_ipc.log
timeout 2400 python -m pytest tests -m gpu -x -q -rs --durations=8 --ignore=tests/test_ipc_multiprocess.py > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest.log
for c in cfg2 cfg3 cfg5; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_$c.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]);r=d['roofline'];o=d['other_policy']
print('$c', d['value'], 'ovh', d['abft_overhead_pct'], 'both', o['abft_overhead_pct'], 'k1', r['k1_ms'], 'k1u', r['k1_unprotected_ms'], 'chk', r['check_ms_per_sweep'], 'frac', r['frac'], d['clocks'])"; done
