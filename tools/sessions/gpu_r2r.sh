#!/bin/bash
# Session R: uniform-kernel register budget A/B (launch bounds 5/6/7 CTAs per
# SM; a1 from global memory so ptxas keeps it in registers).
OUT=gpurun_out/r2r
mkdir -p $OUT
for nnz in 3728 12000; do
  docs=$(( 1300000000 / nnz ))
  AB_NNZ=$nnz AB_DOCS=$docs AB_KS=500,200 AB_REPS=3 AB_ARMS='[{"uniform_2u":2,"uniform_variant":6},{"uniform_2u":2,"uniform_variant":5},{"uniform_2u":2,"uniform_variant":7},{"uniform_2u":2,"uniform_variant":15}]' timeout 600 python tools/ab_uniform.py >> $OUT/regs_ab.jsonl 2>> $OUT/regs_ab.err
done
echo done > $OUT/DONE
