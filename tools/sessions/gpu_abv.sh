#!/bin/bash
# Variant builds: copy the tree to _abv/<name>/, patch, build there (python -c "from paper_1205_2958_b200 import _build; _build.build()")
# Sketch-kernel variants built under _abv/v*/ and the reference build under _ab/, same box.
mkdir -p gpurun_out/abv
rm -f gpurun_out/abv/tune.txt
G='[{"J":8,"TPB":64,"TILE":1024},{"J":8,"TPB":64,"TILE":1280}]'
G4='[{"J":2,"TPB":256,"TILE":4096}]'
for d in $(ls -d _ab _abv/* 2>/dev/null); do
  (cd $d && TUNE_GRID="$G" TUNE_DOCS=200000 python tools/tune.py; TUNE_SCHEMES=4u-bit TUNE_GRID="$G4" TUNE_DOCS=50000 python tools/tune.py) | sed "s|^|$d |" >> gpurun_out/abv/tune.txt 2>&1
done
