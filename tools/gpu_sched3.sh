# schedule A/B: cfg3 forced pipelined with z-chunks 4 / 2 / 1, cfg4 forced pipelined
for zc in auto 2 1; do
  if [ $zc = auto ]; then unset ABFT_ZCHUNK; else export ABFT_ZCHUNK=$zc; fi
  echo "== cfg3 zchunk=$zc"; ABFT_PIPELINE=1 timeout 600 python tools/exp_sched.py cfg3 5 20 2>&1 | grep -v Warn
done
unset ABFT_ZCHUNK
echo "== cfg4"; ABFT_PIPELINE=1 timeout 900 python tools/exp_sched.py cfg4 3 10 2>&1 | grep -v Warn
