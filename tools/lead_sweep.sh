# schedule lead of warp 0 in phase A (cost units; HX_LEAD): controller overlap
for L in 600 1200 2200 3000 6000 100000; do echo -n "lead $L: "; HX_LEAD=$L python tools/quick_rate.py 1; done
