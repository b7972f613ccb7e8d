# task-start alignment of the staggered copy (HX_ALIGN slots; 0 = none)
for c in 1 2; do
for rep in 1 2; do
for a in 0 16 32; do
  HX_ALIGN=$a timeout 120 python tools/quick_rate.py $c 2>&1 | tail -1 | sed "s/^/cfg$c align=$a /"
done; done; done
