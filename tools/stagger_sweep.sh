# A/B of the bank-staggered stream tasks (HX_STAGGER="pmaxA,pmaxT,lmin"; 0,0 = off) with tools/quick_rate.py
for c in 1 2; do
for v in "0,0,4" "15,1,4" "15,1,2" "15,1,8" "7,1,4" "15,2,4" "10,1,4" "0,0,4" "15,1,4" "15,1,3" "15,1,6"; do
  HX_STAGGER=$v timeout 120 python tools/quick_rate.py $c 2>&1 | tail -1 | sed "s/^/cfg$c stagger=$v /"
done; done
