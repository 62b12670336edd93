import os, sys, time, tempfile, ctypes as C
sys.path.insert(0, '/root/repo')
os.environ['BBMH_OPT_TRACE'] = '1'
from oracle import oracle as O
from paper_1205_2958_b200 import bbmh
R = O.ref(); L = R.lib
L.bbmh_synth_classification.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_uint64, C.c_int32]
td = tempfile.mkdtemp(); corpus = td + '/c1.bbcv'
L.bbmh_synth_classification(corpus.encode(), 20000, 1 << 24, 3700 / (1 << 24), 0.3, 0.0, 1, 1)
lib = bbmh.lib()
lib.bbmh_vw_project_file.argtypes = [C.c_char_p, C.c_char_p, C.c_uint32, C.c_uint64]
for i in range(2):
    t = time.perf_counter()
    lib.bbmh_vw_project_file(corpus.encode(), (td + '/vg.txt').encode(), 1 << 20, 3)
    print("CALL", i, time.perf_counter() - t, os.path.getsize(td + '/vg.txt'), file=sys.stderr, flush=True)
