set -x
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/tests_final.log 2>&1; tail -2 gpurun_out/tests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-200
timeout 600 python bench.py --config cfg5 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_cfg5.log 2>&1
timeout 300 python bench.py --config cfg3 --steps 200 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_cfg3.log 2>&1
timeout 300 python bench.py --config cfg2 --steps 100 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_cfg2.log 2>&1
B="python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e"
timeout 600 $B > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1
N="--set full --clock-control none --import-source on --kernel-name-base mangled -c 1"
timeout 300 ncu $N -k regex:k1_sweepIfLi4ELi2ELi0E -s 2 -o gpurun_out/k1_lazy $B > gpurun_out/ncu_a.log 2>&1
timeout 300 ncu $N -k regex:k1_sweepIfLi4ELi1ELi0E -s 2 -o gpurun_out/k1_both $B > gpurun_out/ncu_b.log 2>&1
timeout 300 ncu $N -k regex:k1_sweepIfLi4ELi0ELi0E -s 2 -o gpurun_out/k1_none $B > gpurun_out/ncu_c.log 2>&1
timeout 300 ncu $N -k regex:k2_check -s 4 -o gpurun_out/k2 $B > gpurun_out/ncu_d.log 2>&1
timeout 300 ncu $N -k regex:k3_lazy -s 4 -o gpurun_out/k3 $B > gpurun_out/ncu_e.log 2>&1
timeout 900 python campaign.py --reps 100 --out gpurun_out/campaign.json > gpurun_out/campaign.log 2>&1
ls gpurun_out
