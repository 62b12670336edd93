#!/bin/bash
# Session U: uniform 2U loop shape -- id-major with one two-input min per
# evaluation (the lane-split kernel's shape, which reaches 0.85 at k = 32)
# against the min3 tree; the 4U-bit uniform kernel against the persistent one
# across k (the persistent shapes dip at k = 300).
OUT=gpurun_out/r2u
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for nnz in 3728 12000; do
  docs=$(( 1300000000 / nnz ))
  AB_NNZ=$nnz AB_DOCS=$docs AB_KS=500,200,64 AB_REPS=3 AB_ARMS='[{"uniform_2u":2,"uniform_variant":0},{"uniform_2u":2,"uniform_variant":1}]' timeout 600 python tools/ab_uniform.py >> $OUT/shape_ab.jsonl 2>> $OUT/shape_ab.err
done
AB_SCHEME=4u-bit AB_DOCS=60000 AB_KS=40,48,64,96,128,160,250,300,400,512,600,800,1000 AB_REPS=2 timeout 1200 python tools/ab_uniform.py > $OUT/u4_ks.jsonl 2> $OUT/u4_ks.err
echo done > $OUT/DONE
