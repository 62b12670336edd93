#!/bin/bash
# Round-2 session C: dynamic document tickets in the persistent sketch kernel
# (A/B against round-robin), residency and occupancy with them, GPU tests.
OUT=gpurun_out/r2c
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
G='[{"J":0,"TILE":0,"DYN":0},{"J":0,"TILE":0,"DYN":1},{"J":0,"TILE":0,"DYN":0},{"J":0,"TILE":0,"DYN":1}]'
GC='[{"J":0,"TILE":0,"DYN":1,"SMEM_CAP":1},{"J":0,"TILE":0,"DYN":1,"SMEM_CAP":0},{"J":0,"TILE":0,"DYN":1,"SMEM_CAP":1},{"J":0,"TILE":0,"DYN":1,"SMEM_CAP":0}]'
for K in 500 300 200 64; do
  TUNE_K=$K TUNE_GRID="$G" TUNE_DOCS=200000 TUNE_SCHEMES=2u timeout 300 python tools/tune.py >> $OUT/dyn.jsonl 2>> $OUT/dyn.err
  TUNE_K=$K TUNE_GRID="$G" TUNE_DOCS=50000 TUNE_SCHEMES=4u-bit timeout 300 python tools/tune.py >> $OUT/dyn.jsonl 2>> $OUT/dyn.err
done
TUNE_K=200 TUNE_GRID="$GC" TUNE_DOCS=200000 TUNE_SCHEMES=2u timeout 300 python tools/tune.py >> $OUT/dyn.jsonl 2>> $OUT/dyn.err
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I paper_1205_2958_b200/csrc tools/residency_probe.cu \
  paper_1205_2958_b200/csrc/perm.cu paper_1205_2958_b200/csrc/options.cpp -o /tmp/residency_probe > $OUT/probe_build.log 2>&1
timeout 120 /tmp/residency_probe 350000 > $OUT/residency.jsonl 2>&1
timeout 600 ncu --section Occupancy --section LaunchStats --section SpeedOfLight \
    --metrics sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:sketch_kernel -s 2 -c 2 --csv \
    python bench.py --docs 100000 --steps 1 --warmup 2 --schemes 2u,4u-bit --e2e-steps 1 --no-cpu > $OUT/ncu_occ.csv 2> $OUT/ncu_occ.err
timeout 900 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest gpu exit $?" >> $OUT/pytest_gpu.log
echo done > $OUT/DONE
