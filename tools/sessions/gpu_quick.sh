#!/bin/bash
# Quick iteration session: tests + smoke + intpeak + 1-GPU bench (+ optional ncu on the top kernel).
TAG=${1:-q}
NCU=${2:-0}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest gpu exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 120 python tools/intpeak.py $OUT/int_peaks.json > $OUT/intpeak.log 2>&1
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
if [ "$NCU" = "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --docs 50000 --steps 2 --warmup 1 --e2e-steps 1 --no-cpu > $OUT/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sketch_kernel -s 2 -c 1 \
    -o $OUT/prof_2u python bench.py --docs 20000 --steps 1 --warmup 2 --schemes 2u --e2e-steps 1 --no-cpu > $OUT/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sketch_kernel -s 2 -c 1 \
    -o $OUT/prof_4u python bench.py --docs 20000 --steps 1 --warmup 2 --schemes 4u-bit --e2e-steps 1 --no-cpu > $OUT/ncu_full4.log 2>&1
fi
echo done > $OUT/DONE
