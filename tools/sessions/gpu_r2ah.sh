#!/bin/bash
# Session AH: uniform 2U kernel with 16 ids per lane per step (loads at the top
# of the step, no register double buffer) against the shipped 8-id step.
OUT=gpurun_out/r2ah
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for nnz in 3728 12000; do
  docs=$(( 1300000000 / nnz ))
  AB_NNZ=$nnz AB_DOCS=$docs AB_KS=500,200,64 AB_REPS=3 AB_ARMS='[{"uniform_2u":2,"uniform_variant":0},{"uniform_2u":2,"uniform_variant":1}]' timeout 600 python tools/ab_uniform.py >> $OUT/ab16.jsonl 2>> $OUT/ab16.err
done
echo done > $OUT/DONE
