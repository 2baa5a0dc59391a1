"""Dev probe: time the tcgen05 assignment filter alone (use under ncu).
usage: python scripts/tc_bench.py [n] [k] [hh_only]"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2107_06876_b200 as lcn

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
hh = int(sys.argv[3]) if len(sys.argv) > 3 else 0
d = 128
ctx = lcn.Context(0)
lib = lcn.library()
lib.lcn_debug_tc_scores.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t, C.c_void_p, C.c_size_t, C.c_int,
                                    C.c_void_p]
r = np.random.default_rng(0)
x = r.standard_normal((n, d)).astype(np.float32)
c = x[r.choice(n, k, replace=False)].astype(np.float64)
acc = np.zeros(128 * 64, np.float32)
for _ in range(2):
    st = lib.lcn_debug_tc_scores(ctx.h, x.ctypes.data, n, d, c.ctypes.data, k, hh, acc.ctypes.data)
    assert st == 0, st
print("ok")
