# A/B of the in-tree build against tools/explib/libabft_old.so (interleaved
# step(K) device times, medians; tools/exp_lib_ab.py) on cfg2, cfg3, cfg4
for c in cfg2 cfg3; do timeout 600 python tools/exp_lib_ab.py $c base old 7 2>&1 | grep -v Warn; done
timeout 900 python tools/exp_lib_ab.py cfg4 base old 5 2>&1 | grep -v Warn
