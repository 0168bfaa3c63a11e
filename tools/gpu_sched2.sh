for z in 13 4 2 1; do echo "== cfg3 zchunk $z"; ABFT_ZCHUNK=$z timeout 600 python tools/exp_sched.py cfg3 5 20 2>&1 | grep -v "_nog\|_pdl\|_lo" | tail -6; done
for z in 8 4; do echo "== cfg4 zchunk $z"; ABFT_ZCHUNK=$z timeout 600 python tools/exp_sched.py cfg4 3 20 2>&1 | grep -v "_nog\|_pdl\|_lo" | tail -6; done
