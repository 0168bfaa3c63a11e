# cfg5 (per-GPU slab 2048x2048x128 fp64, 27-point, offline) -- bench line, then
# the launch list and one ncu --set full capture of the fp64 K1, each after
# the same command exited 0 without ncu
B="python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu --no-e2e"
mkdir -p gpurun_out/c5
timeout 600 python bench.py --config cfg5 --steps 20 --warmup 5 --no-cpu > gpurun_out/c5/bench_cfg5.log 2>&1
timeout 600 $B > gpurun_out/c5/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5/launches.csv $B > gpurun_out/c5/ncu_list.log 2>&1
N="--set full --clock-control none --kernel-name-base mangled -c 1"
timeout 400 ncu $N --import-source on -k regex:k1_sweepId -s 6 -o gpurun_out/c5/k1_cfg5 $B > gpurun_out/c5/ncu_k1.log 2>&1
timeout 400 ncu --page raw --csv -i gpurun_out/c5/k1_cfg5.ncu-rep > gpurun_out/c5/k1_cfg5_raw.csv 2>&1
du -sh gpurun_out/c5; ls -la gpurun_out/c5
