"""One device-resident sketch launch (for ncu): SCHEME K DOCS from the env."""
import os
import sys

import torch

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1205_2958_b200 import bbmh  # noqa: E402

scheme = os.environ.get("SCHEME", "2u")
k = int(os.environ.get("K", "1"))
n = int(os.environ.get("DOCS", "200000"))
sid, dim = bench.SCHEMES[scheme]
dev = torch.device("cuda", 0)
d_rp, d_idx = bench.make_corpus_device(torch, n, bench.NNZ, bench.D_WEBSPAM, 5, dev)
cb = (k * 8 + 7) // 8
d_codes = torch.empty(n * cb, dtype=torch.uint8, device=dev)
f = bbmh.Family(sid, dim, k, 42)
st = torch.cuda.current_stream()
for _ in range(3):
    f.sketch_csr_device(d_rp.data_ptr(), d_idx.data_ptr(), n, 8, d_codes.data_ptr(), stream=st.cuda_stream)
torch.cuda.synchronize()
print("done", scheme, k, n)
