# ncu --set full of one cfg3 K1 launch unprotected (NONE) and one protected (LAZY)
mkdir -p /tmp/nc
for s in 10 35; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_sweep -s $s -c 1 -o /tmp/nc/k1_cfg3_s$s python tools/exp_small.py cfg3 > gpurun_out/ncu_cfg3_s$s.log 2>&1
  python tools/ncu_summary.py /tmp/nc/k1_cfg3_s$s.ncu-rep > gpurun_out/k1_cfg3_s$s.txt 2>&1
  python tools/ncu_summary.py --sass /tmp/nc/k1_cfg3_s$s.ncu-rep >> gpurun_out/k1_cfg3_s$s.txt 2>&1
  cp /tmp/nc/k1_cfg3_s$s.ncu-rep gpurun_out/
done
