# round measurements: smoke, bench lines (cfg4 headline with e2e + cpu baseline,
# cfg5 slab, cfg3, cfg2), the reference arm, launch lists and ncu --set full
# captures of the top kernels (each after its command ran clean without ncu),
# the unprotected K1 beside the protected one
mkdir -p /tmp/nc
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log | cut -c1-200
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo bench4_rc=$?
for c in cfg5 cfg3 cfg2; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_${c}_rc=$?; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
for c in cfg4 cfg5 cfg3 cfg2; do python - <<PY
import json
d=json.loads(open("gpurun_out/bench_$c.json").read().strip().splitlines()[-1])
r=d["roofline"]; o=d["other_policy"]
print("$c", d["value"], "ovh", d["abft_overhead_pct"], "flips", d["abft_overhead_with_flips_pct"], "other", o["abft_overhead_pct"], "prot", d["error_free_protected_gcells"], "unprot", d["unprotected_gcells"], "k1", r["k1_ms"], "k1u", r["k1_unprotected_ms"], "chk", r["check_ms_per_sweep"], "frac", r["frac"], "e2e", (d.get("e2e") or {}).get("value"), d["clocks"])
PY
done
tail -c 600 gpurun_out/bench_ref.json
B4="python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e"
B5="python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv $B4 > /dev/null 2>&1; echo l4=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv $B5 > /dev/null 2>&1; echo l5=$?
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:k1_sweep -s 2 -c 1 -o /tmp/nc/k1_cfg4_lazy $B4 > gpurun_out/ncu_k1_4.log 2>&1; echo n4=$?
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:k2_check -s 2 -c 1 -o /tmp/nc/k2_cfg4_lazy $B4 > gpurun_out/ncu_k2_4.log 2>&1; echo n42=$?
timeout 600 ncu -f --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:_ZN4abft8k1_sweepIfLi4ELi0ELi0E -s 2 -c 1 -o /tmp/nc/k1_cfg4_none $B4 > gpurun_out/ncu_k1_4n.log 2>&1; echo n4n=$?
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:k1_sweep -s 30 -c 1 -o /tmp/nc/k1_cfg5 $B5 > gpurun_out/ncu_k1_5.log 2>&1; echo n5=$?
for r in k1_cfg4_lazy k1_cfg4_none k2_cfg4_lazy k1_cfg5; do python tools/ncu_summary.py /tmp/nc/$r.ncu-rep > gpurun_out/$r.txt 2>&1; python tools/ncu_summary.py --sass /tmp/nc/$r.ncu-rep >> gpurun_out/$r.txt 2>&1; cp /tmp/nc/$r.ncu-rep gpurun_out/; done
python tools/ncu_summary.py --launches gpurun_out/launches_cfg4.csv > gpurun_out/launches_summary.txt
python tools/ncu_summary.py --launches gpurun_out/launches_cfg5.csv >> gpurun_out/launches_summary.txt
head -30 gpurun_out/launches_summary.txt
