# schedule cost constants re-swept with the bank-staggered layout (HX_COSTS="rowT,taskT,rowA,taskA")
for c in 1 2; do
for v in "5,64,5,64" "4,64,5,64" "7,64,5,64" "5,64,3,64" "5,64,8,64" "5,32,5,32" "5,96,5,96" "5,64,5,64"; do
  HX_COSTS=$v timeout 120 python tools/quick_rate.py $c 2>&1 | tail -1 | sed "s/^/cfg$c costs=$v /"
done; done
for l in 2000 3000 4500; do HX_LEAD=$l timeout 120 python tools/quick_rate.py 1 2>&1 | tail -1 | sed "s/^/cfg1 lead=$l /"; done
