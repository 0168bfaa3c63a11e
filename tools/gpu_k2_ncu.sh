# ncu --set full of one K2 launch: cfg4 LAZY (bench) and cfg3 LAZY serial (exp_small)
mkdir -p /tmp/nc
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:k2_check -s 2 -c 1 -o /tmp/nc/k2_cfg4 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo r4=$?
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:k2_check -s 10 -c 1 -o /tmp/nc/k2_cfg3 python tools/exp_small.py cfg3 > /dev/null 2>&1; echo r3=$?
for r in k2_cfg4 k2_cfg3; do python tools/ncu_summary.py /tmp/nc/$r.ncu-rep > gpurun_out/$r.txt 2>&1; python tools/ncu_summary.py --sass /tmp/nc/$r.ncu-rep >> gpurun_out/$r.txt 2>&1; cp /tmp/nc/$r.ncu-rep gpurun_out/; done
