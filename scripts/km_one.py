"""Dev probe: one lloyd (k-means++ seeding + 10 iterations) on 2e6 x 128
configs[3]-like mixture points (for ncu captures of the seeding kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2107_06876_b200 as lcn
N = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
d = 128
rng = np.random.default_rng(5)
means = rng.standard_normal((1000, d))
x = (means[rng.integers(0, 1000, N)] + 0.5 * rng.standard_normal((N, d))).astype(np.float32).astype(np.float64)
ctx = lcn.Context(0)
c, a = lcn.lloyd(ctx, x, K, 1, 7)
print("ok", a[:4])
