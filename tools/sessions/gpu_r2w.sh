#!/bin/bash
# Session W: GPU tests after the small-k routing (2U 16 < k < 32 on the
# device: both kernels; 4U 16 < k <= 32 uniform), k sweep, sanitizers.
OUT=gpurun_out/r2w
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest gpu exit $?" >> $OUT/pytest_gpu.log
timeout 900 python tools/bench_configs.py --only ksweep --out $OUT/ksweep.jsonl > $OUT/ksweep.log 2>&1
bash tools/gpu_sanitize.sh r2w/san
echo done > $OUT/DONE
