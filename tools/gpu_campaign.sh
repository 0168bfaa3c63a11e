# the fault-injection campaign (E1, E3) and its markdown summary
timeout 1800 python campaign.py --exp e1,e3 --reps 20 --out gpurun_out/campaign.json > gpurun_out/campaign.log 2>&1; echo campaign_rc=$?
python tools/campaign_summary.py gpurun_out/campaign.json > gpurun_out/campaign_summary.md 2>&1
# A/B of K2 CTA widths (experiment builds in tools/explib)
for c in cfg3 cfg4; do timeout 600 python tools/exp_lib_ab.py $c base ct256 ct256ku2 5 2>&1 | grep -v Warn; done
