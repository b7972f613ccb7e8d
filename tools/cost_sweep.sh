# schedule cost model (HX_COSTS = rowA,taskA,rowB,taskB in nnz units; A = A^T's
# rows in phase A, B = A's rows in phase B) against configs[1] / [2]
for c in "5,64,5,64" "7,64,7,64" "10,64,10,64" "14,64,14,64" "5,64,10,64" "10,64,5,64" "20,64,20,64"; do
  for g in 1 2; do echo -n "$c cfg$g: "; HX_COSTS=$c python tools/quick_rate.py $g; done
done
