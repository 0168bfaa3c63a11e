# the bit-position experiment E2 of campaign.py and its summary
timeout 1500 python campaign.py --exp e2 --reps 10 --out gpurun_out/campaign_e2.json > gpurun_out/campaign_e2.log 2>&1; echo campaign_rc=$?
python tools/campaign_summary.py gpurun_out/campaign_e2.json > gpurun_out/campaign_e2_summary.md 2>&1
tail -3 gpurun_out/campaign_e2.log
