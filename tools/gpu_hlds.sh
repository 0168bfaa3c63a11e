# fp64 x-halo from shared memory (ABFT_HALO_LDS=1 experiment build): A/B and ncu of the cfg5 K1
timeout 900 python tools/exp_lib_ab.py cfg5 base hlds 3 2>&1 | grep -v Warn
mkdir -p /tmp/nc
B5="python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu --no-e2e"
ABFT_LIB=$PWD/tools/explib/libabft_hlds.so timeout 600 ncu --set full --clock-control none -k regex:k1_sweep -s 30 -c 1 -o /tmp/nc/k1_cfg5_hlds $B5 > /dev/null 2>&1; echo n5=$?
python tools/ncu_summary.py /tmp/nc/k1_cfg5_hlds.ncu-rep > gpurun_out/k1_cfg5_hlds.txt 2>&1; python tools/ncu_summary.py --sass /tmp/nc/k1_cfg5_hlds.ncu-rep >> gpurun_out/k1_cfg5_hlds.txt 2>&1
grep -E "duration|inst_executed|issue_active|wavefronts|SHFL|FSEL|LDS|stall" gpurun_out/k1_cfg5_hlds.txt
