set -x
mkdir -p /tmp/nc
B5="python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_check -s 40 -c 1 -o /tmp/nc/k2_cfg5 $B5 > gpurun_out/ncu_k2_5.log 2>&1
B4="python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_check -s 10 -c 1 -o /tmp/nc/k2_cfg4_lazy $B4 > gpurun_out/ncu_k2_4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_check -s 20 -c 1 -o /tmp/nc/k2_cfg4_both $B4 --policy both > gpurun_out/ncu_k2_4b.log 2>&1
ls -la /tmp/nc
for r in k2_cfg5 k2_cfg4_lazy k2_cfg4_both; do python tools/ncu_summary.py /tmp/nc/$r.ncu-rep > gpurun_out/$r.txt 2>&1; python tools/ncu_summary.py --sass /tmp/nc/$r.ncu-rep >> gpurun_out/$r.txt 2>&1; ncu -i /tmp/nc/$r.ncu-rep --page source --csv > gpurun_out/${r}_source.csv 2>/dev/null; done
cp /tmp/nc/k2_cfg4_lazy.ncu-rep gpurun_out/
ls -la gpurun_out
