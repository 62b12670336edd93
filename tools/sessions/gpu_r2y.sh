#!/bin/bash
# Session Y: grouped lane-split 2U kernel (gsplit.cu) against the uniform
# kernel and the persistent kernel, codes and minima compared.
OUT=gpurun_out/r2y
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for nnz in 3728 12000 1500; do
  docs=$(( 1300000000 / nnz ))
  AB_NNZ=$nnz AB_DOCS=$docs AB_KS=500,200,100,64,33 AB_BS=8,5 AB_REPS=3 AB_ARMS='[{"uniform_2u":2,"gsplit_2u":0},{"uniform_2u":2,"gsplit_2u":1}]' timeout 900 python tools/ab_uniform.py >> $OUT/gsplit_ab.jsonl 2>> $OUT/gsplit_ab.err
done
echo done > $OUT/DONE
