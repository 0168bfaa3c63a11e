set -x
mkdir -p /tmp/nc
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg2 or tile or lazy or ragged or box27 or cfg5 or slab" > gpurun_out/pytest_k1.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest_k1.log
for i in 1 2; do timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_cfg4_$i.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg4_$i.json').read().strip().splitlines()[-1]);r=d['roofline'];o=d['other_policy']
print('cfg4', d['value'], 'ovh', d['abft_overhead_pct'], 'both', o['abft_overhead_pct'], 'k1L', r['k1_ms'], 'k1B', o['k1_ms'], 'k1u', r['k1_unprotected_ms'], 'chk', r['check_ms_per_sweep'], o['check_ms_per_sweep'], d['clocks'])"; done
B4="python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e"
timeout 600 ncu --set full --clock-control none -k regex:k1_sweep -s 2 -c 1 -o /tmp/nc/k1_lazy $B4 > gpurun_out/ncu_a.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k1_sweep -s 70 -c 1 -o /tmp/nc/k1_x $B4 > gpurun_out/ncu_b.log 2>&1
for r in k1_lazy k1_x; do python tools/ncu_summary.py /tmp/nc/$r.ncu-rep > gpurun_out/$r.txt 2>&1; ncu -i /tmp/nc/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/${r}_src.csv 2>/dev/null; done
head -3 gpurun_out/k1_lazy.txt gpurun_out/k1_x.txt
