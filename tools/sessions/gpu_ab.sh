#!/bin/bash
# Reference build: rm -rf _ab && mkdir _ab && git archive <commit> | tar -x -C _ab && (cd _ab && python -c "from paper_1205_2958_b200 import _build; _build.build()")
# A/B of the sketch kernel: a reference build under _ab/ (git archive of an older
# commit, built there) against the working tree, same box, same process order.
mkdir -p gpurun_out/ab
rm -f gpurun_out/ab/tune.txt
G4='[{"J":2,"TPB":256,"TILE":4096}]'
for i in 1 2; do
  (cd _ab && TUNE_GRID="$(cat ../tools/grid_2u.json)" TUNE_DOCS=200000 python tools/tune.py) | sed 's/^/old /' >> gpurun_out/ab/tune.txt 2>&1
  TUNE_GRID="$(cat tools/grid_2u.json)" TUNE_DOCS=200000 python tools/tune.py | sed 's/^/new /' >> gpurun_out/ab/tune.txt 2>&1
  (cd _ab && TUNE_SCHEMES=4u-bit TUNE_GRID="$G4" TUNE_DOCS=50000 python tools/tune.py) | sed 's/^/old /' >> gpurun_out/ab/tune.txt 2>&1
  TUNE_SCHEMES=4u-bit TUNE_GRID="$G4" TUNE_DOCS=50000 python tools/tune.py | sed 's/^/new /' >> gpurun_out/ab/tune.txt 2>&1
done
