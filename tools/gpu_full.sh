# full GPU pass: tests, bench, launch list, ncu captures of K1 (protected, unprotected) and K2
set -x
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/tests.log 2>&1; tail -25 gpurun_out/tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -3 gpurun_out/bench.log
B="python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e"
timeout 600 $B > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_sweep -s 4 -c 1 -o gpurun_out/k1prot $B > gpurun_out/ncu_k1p.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_sweep -s 17 -c 1 -o gpurun_out/k1unprot $B > gpurun_out/ncu_k1u.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_check -s 4 -c 1 -o gpurun_out/k2 $B > gpurun_out/ncu_k2.log 2>&1
ls -la gpurun_out
