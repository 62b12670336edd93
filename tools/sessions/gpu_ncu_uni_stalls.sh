#!/bin/bash
# ncu --set full of the coefficient-uniform 2U kernel (stall reasons, source
# page) at the C2 shape, k = 500 and 64, forced on (uniform_2u = 2).
OUT=gpurun_out/${1:-us}
mkdir -p $OUT
for k in ${NCU_KS:-500 64}; do
ONCE_UNIFORM=2 ONCE_K=$k ONCE_DOCS=${ONCE_DOCS:-60000} timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:sketch_uniform -s 1 -c 1 -o $OUT/uni_k$k python tools/uniform_once.py > $OUT/ncu_k$k.log 2>&1
done
echo done > $OUT/DONE
