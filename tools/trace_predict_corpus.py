import sys, os, time, json, ctypes as C, numpy as np, tempfile
sys.path.insert(0, '/root/repo')
os.environ['BBMH_OPT_TRACE'] = '1'
from oracle import oracle as O
from paper_1205_2958_b200 import bbmh
R = O.ref(); L = R.lib
L.bbmh_synth_classification.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_uint64, C.c_int32]
td = tempfile.mkdtemp(); corpus = td + '/c1.bbcv'
L.bbmh_synth_classification(corpus.encode(), 20000, 1 << 24, 3700 / (1 << 24), 0.3, 0.0, 1, 1)
k, b = 200, 8
w = np.random.default_rng(0).standard_normal(k << b)
model = td + '/m.bblm'
open(model, 'wb').write(b"BBLM" + (k << b).to_bytes(8, "little") + bytes([0, 0]) + w.astype("<f8").tobytes())
f = bbmh.Family(1, 1 << 24, k, 42)
for i in range(2):
    t = time.perf_counter(); st = {}
    f.predict_corpus(b, model, corpus, td + '/g.tsv', 16, stats=st)
    print("CALL", i, time.perf_counter() - t, st, file=sys.stderr, flush=True)
