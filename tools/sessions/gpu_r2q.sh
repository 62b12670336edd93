#!/bin/bash
# Session Q: full validation of the round-2 product (tests, smoke, default
# bench with every scheme and the CPU reference, reference arm), then ncu:
# a full-size capture of the C2 2U launch (now the uniform kernel) for the
# traffic figure, the bench's launch list.
OUT=gpurun_out/r2q
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 900 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest gpu exit $?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref exit $?" >> $OUT/bench_ref.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sketch_uniform -s 3 -c 1 \
    -o $OUT/prof_2u_full python bench.py --steps 1 --warmup 3 --schemes 2u --e2e-steps 1 --no-cpu > $OUT/ncu_2u.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu > $OUT/launches.log 2>&1
echo done > $OUT/DONE
