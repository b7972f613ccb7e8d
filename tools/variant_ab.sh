# A/B of build variants (tools/variant.sh) with tools/quick_rate.py: VARIANTS="a b" CFGS="1 2" bash tools/variant_ab.sh
for c in ${CFGS:-1 2}; do
for rep in 1 2; do
for v in ${VARIANTS}; do
  HPLP_GPU_LIB=build_variants/$v/libhplp_gpu.so timeout 120 python tools/quick_rate.py $c 2>&1 | tail -1 | sed "s|^|cfg$c $v |"
done; done; done
