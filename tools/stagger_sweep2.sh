# HX_STAGGER re-swept on the aligned layout (HX_ALIGN=32)
for c in 1 2; do
for v in "15,1,4" "15,0,4" "15,2,4" "15,3,4" "7,1,4" "15,1,8"; do
  HX_STAGGER=$v timeout 120 python tools/quick_rate.py $c 2>&1 | tail -1 | sed "s/^/cfg$c stagger=$v /"
done; done
