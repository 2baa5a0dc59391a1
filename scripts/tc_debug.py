"""Dev probe: tcgen05 filter accumulators vs numpy (first tile)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2107_06876_b200 as lcn
lib = lcn.library()
lib.lcn_debug_tc_scores.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]
ctx = lcn.Context(0)
r = np.random.default_rng(1)
n, d, k = 128, 128, 64
x = r.standard_normal((n, d)).astype(np.float32)
c = r.standard_normal((k, d))
def hi(a):
    return (a.astype(np.float32).view(np.uint32) & np.uint32(0xffffe000)).view(np.float32)
for hh in (1, 0):
    acc = np.zeros((128, 64), np.float32)
    st = lib.lcn_debug_tc_scores(ctx.h, x.ctypes.data, n, d, c.ctypes.data, k, hh, acc.ctypes.data)
    print("status", st)
    cf = c.astype(np.float32)
    ref_hh = hi(x).astype(np.float64) @ hi(cf).astype(np.float64).T
    ref = x.astype(np.float64) @ cf.astype(np.float64).T
    want = ref_hh if hh else ref
    err = np.abs(acc - want)
    print("hh_only" if hh else "3xtf32", "max err", err.max(), "rel", (err / (np.abs(want) + 1e-6)).max())
    print(" acc[0,:6]", acc[0, :6]); print(" ref[0,:6]", want[0, :6].astype(np.float32))
    print(" acc[1,:6]", acc[1, :6]); print(" ref[1,:6]", want[1, :6].astype(np.float32))
    # try to identify permutations
    if err.max() > 1e-2:
        best = np.argmin(np.abs(acc[0][None, :] - want[:, :]).sum(1)) if False else None
        for i in range(3):
            j = np.argmin(np.abs(want - acc[i, 0]).ravel())
            print("  acc[%d,0] matches ref flat idx" % i, np.unravel_index(j, want.shape))
np.savez("gpurun_out/tc_debug.npz", x=x, c=c, acc=acc)
