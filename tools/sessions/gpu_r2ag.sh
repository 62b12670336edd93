#!/bin/bash
# Session AG: small 4U-bit batches (C5 sizes) through the uniform 4U kernel
# (forced) against the persistent kernel, device-resident, k = 500.
OUT=gpurun_out/r2ag
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for n in 64 256 1024 2048 4096; do
  AB_SCHEME=4u-bit AB_DOCS=$n AB_KS=500,200 AB_REPS=20 timeout 300 python tools/ab_uniform.py >> $OUT/u4_small.jsonl 2>> $OUT/u4_small.err
done
echo done > $OUT/DONE
