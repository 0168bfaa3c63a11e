# ncu --set full of one cfg3 K2 (lazy, serial) and one K3, plus cfg4 K2 (lazy)
mkdir -p /tmp/nc
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_check -s 10 -c 1 -o /tmp/nc/k2_cfg3 python tools/exp_small.py cfg3 > gpurun_out/ncu_k2_cfg3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k3_lazy -s 10 -c 1 -o /tmp/nc/k3_cfg3 python tools/exp_small.py cfg3 > gpurun_out/ncu_k3_cfg3.log 2>&1
for r in k2_cfg3 k3_cfg3; do python tools/ncu_summary.py /tmp/nc/$r.ncu-rep > gpurun_out/$r.txt 2>&1; python tools/ncu_summary.py --sass /tmp/nc/$r.ncu-rep >> gpurun_out/$r.txt 2>&1; cp /tmp/nc/$r.ncu-rep gpurun_out/; done
