#!/bin/bash
# Session AE: stall reasons of the persistent 4U-bit kernel at k = 500 (C2 docs).
OUT=gpurun_out/r2ae
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
cat > /tmp/once4.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_1205_2958_b200 import bbmh
n, k = 60000, int(os.environ.get("K", "500"))
bbmh.set_option("uniform_4u", 0)
d_rp, d_idx = bench.make_corpus_device(torch, n, bench.NNZ, bench.D_WEBSPAM, 1, torch.device("cuda", 0))
f = bbmh.Family(3, bench.D_WEBSPAM, k, bench.SEED)
codes = torch.zeros(n * k, dtype=torch.uint8, device="cuda")
for _ in range(2):
    f.sketch_csr_device(d_rp.data_ptr(), d_idx.data_ptr(), n, 8, codes.data_ptr(), stream=torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
PY
K=500 timeout 900 ncu --set full --clock-control none --import-source on -k regex:sketch_kernel -s 1 -c 1 -o $OUT/p4_k500 python /tmp/once4.py > $OUT/p4.log 2>&1
echo done > $OUT/DONE
