#!/bin/bash
# One gpurun session: tests, smoke, int peaks, bench, launch list, one full ncu capture.
# Usage (from the repo root, on the GPU box): bash tools/sessions/gpu_session.sh [tag]
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nproc > $OUT/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)|Socket" >> $OUT/nproc.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest gpu exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 120 python tools/intpeak.py $OUT/int_peaks.json > $OUT/intpeak.log 2>&1
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --docs 50000 --steps 2 --warmup 1 --e2e-steps 1 --no-cpu > $OUT/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sketch_kernel -s 2 -c 1 \
    -o $OUT/prof_2u python bench.py --docs 20000 --steps 1 --warmup 2 --schemes 2u --e2e-steps 1 --no-cpu > $OUT/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sketch_kernel -s 2 -c 1 \
    -o $OUT/prof_4u python bench.py --docs 20000 --steps 1 --warmup 2 --schemes 4u-bit --e2e-steps 1 --no-cpu > $OUT/ncu_full4.log 2>&1
echo done > $OUT/DONE
