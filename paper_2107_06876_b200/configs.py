"""Seeded synthetic inputs for the BASELINE.json configs (no public dataset is used).

The paper's EN-DE embeddings and GED graphs are not in this image, so each
config is a seeded Gaussian-mixture stand-in with the shapes, sizes and cost
the config names. Points are drawn in fp32 with numpy's PCG64
(bit-stable across machines) and promoted exactly to fp64 for the solver API,
which is fp64 like the reference (geometry.hpp:14-18).

Seeds follow the reference runner's derivation (runner.cpp:175-180): a base
seed per config, LSH seed = mix_seed(seed, 3) (runner.cpp:256), landmark seed
= mix_seed(seed, 4) (runner.cpp:265).

Squared-L2 configs are normalised by the mean pairwise cost mu (configs[0]
says so; configs[3] must be, or every linear-space kernel value underflows,
SURVEY.md Appendix B.2). The normalisation is carried as lambda_eff =
lambda * mu with cost = raw squared L2, which gives the identical kernel
exp(-C / (mu * lambda)); the reported distance is the solver's distance / mu.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

# Cost kinds (reference geometry.hpp:35-39 order, + documented SqEuclidean).
EUCLIDEAN, NEGATIVE_DOT, COSINE_DERIVED, SQEUCLIDEAN = 0, 1, 2, 3
LANDMARK_KMEANS, LANDMARK_KMEANSPP = 0, 1


def mix_seed(seed: int, salt: int) -> int:
    """runner.cpp:175-180."""
    m = (1 << 64) - 1
    x = (seed ^ ((salt * 0x9E3779B97F4A7C15) & m)) & m
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & m
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & m
    return x ^ (x >> 31)


def mix_seed_array(seeds: np.ndarray, salt: int) -> np.ndarray:
    """mix_seed over a uint64 array (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        x = np.asarray(seeds, np.uint64) ^ np.uint64((salt * 0x9E3779B97F4A7C15) & ((1 << 64) - 1))
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


@dataclasses.dataclass
class Problem:
    name: str
    p: np.ndarray            # n x d float64 (fp32-representable)
    q: np.ndarray            # m x d float64
    cost: int
    lam: float               # lambda the config names
    lam_eff: float           # lambda passed to the solver (lam * mu for normalised sq-L2)
    mu: float                # distance scale (1 unless normalised)
    bands: int
    buckets: int
    kmeans_iters: int
    landmarks: int           # 0 = sparse-only variant
    iters: int
    seed: int

    @property
    def n(self):
        return self.p.shape[0]

    @property
    def m(self):
        return self.q.shape[0]

    @property
    def d(self):
        return self.p.shape[1]

    @property
    def lsh_seed(self):
        return mix_seed(self.seed, 3)

    @property
    def landmark_seed(self):
        return mix_seed(self.seed, 4)

    def marginals(self):
        return np.full(self.n, 1.0 / self.n), np.full(self.m, 1.0 / self.m)


def _mixture(rng, n, d, comps, mean_std, sigma, means=None):
    if means is None:
        means = (rng.standard_normal((comps, d), dtype=np.float32) * np.float32(mean_std))
    lab = rng.integers(0, comps, size=n)
    x = means[lab] + rng.standard_normal((n, d), dtype=np.float32) * np.float32(sigma)
    return x.astype(np.float32), means


def mean_sq_cost(p: np.ndarray, q: np.ndarray) -> float:
    """Mean of ||x - y||^2 over all n*m pairs, closed form, rounded to 12
    significant digits so every machine derives the same lambda_eff."""
    p64, q64 = p.astype(np.float64), q.astype(np.float64)
    mu = (math.fsum(np.einsum("ij,ij->i", p64, p64)) / len(p64)
          + math.fsum(np.einsum("ij,ij->i", q64, q64)) / len(q64)
          - 2.0 * float(np.dot(p64.mean(0), q64.mean(0))))
    return float(f"{mu:.12g}")


def config0(scale: float = 1.0) -> Problem:
    """configs[0]: sparse Sinkhorn, n=m=2000, d=32, one shared 10-component
    mixture (means ~ N(0,4I), sigma=1), sq-L2 / mean, lambda=0.1, 1 x 16 k-means
    LSH, 100 iterations."""
    seed = 1000
    n = max(16, int(2000 * scale))
    rng = np.random.default_rng(seed)
    p, means = _mixture(rng, n, 32, 10, 2.0, 1.0)
    q, _ = _mixture(rng, n, 32, 10, 2.0, 1.0, means)
    mu = mean_sq_cost(p, q)
    return Problem("c0_sparse", p.astype(np.float64), q.astype(np.float64), SQEUCLIDEAN, 0.1, 0.1 * mu, mu,
                   1, 16, 10, 0, 100, seed)


def config1(scale: float = 1.0) -> Problem:
    """configs[1]: LCN, n=m=20000, d=300, unit-normalised 50-component mixture
    (means ~ N(0,I), sigma=0.5: unspecified by the config, recorded here);
    target = source @ R (Haar, QR with sign fix) + N(0, 0.05^2), renormalised.
    L2 cost, lambda=0.05, 200 k-means landmarks, 2 x 128 k-means LSH, 50 iterations."""
    seed = 1001
    n = max(256, int(20000 * scale))
    d = 300
    rng = np.random.default_rng(seed)
    src, _ = _mixture(rng, n, d, 50, 1.0, 0.5)
    src = src / np.linalg.norm(src, axis=1, keepdims=True)
    g = rng.standard_normal((d, d))
    qm, r = np.linalg.qr(g)
    qm = qm * np.sign(np.diag(r))
    tgt = src.astype(np.float64) @ qm + 0.05 * rng.standard_normal((n, d))
    tgt = tgt / np.linalg.norm(tgt, axis=1, keepdims=True)
    p = src.astype(np.float32).astype(np.float64)
    q = tgt.astype(np.float32).astype(np.float64)
    buckets = 128 if scale >= 1.0 else max(4, int(128 * scale))
    l = 200 if scale >= 1.0 else max(8, int(200 * scale))
    return Problem("c1_lcn", p, q, EUCLIDEAN, 0.05, 0.05, 1.0, 2, buckets, 10, l, 50, seed)


def config3(scale: float = 1.0) -> Problem:
    """configs[3]: LCN at scale, n=m=1e6, d=128, one shared 1000-component mixture
    (sigma=0.5, means ~ N(0,I)), sq-L2 / mean, lambda=0.05, 512 k-means landmarks,
    2 x 4096 k-means LSH, 100 iterations. `scale` shrinks n and the bucket count
    together (mean bucket size ~488 points kept)."""
    seed = 1003
    n = max(64, int(1_000_000 * scale))
    rng = np.random.default_rng(seed)
    comps = max(2, int(round(1000 * scale))) if scale < 1.0 else 1000
    p, means = _mixture(rng, n, 128, comps, 1.0, 0.5)
    q, _ = _mixture(rng, n, 128, comps, 1.0, 0.5, means)
    mu = mean_sq_cost(p, q)
    buckets = 4096 if scale >= 1.0 else max(2, int(round(4096 * scale)))
    l = 512 if scale >= 1.0 else min(512, max(8, 2 * n // 100))
    return Problem("c3_lcn", p.astype(np.float64), q.astype(np.float64), SQEUCLIDEAN, 0.05, 0.05 * mu, mu,
                   2, buckets, 10, l, 100, seed)


@dataclasses.dataclass
class Batch:
    """configs[4]: many independent small LCN problems, flattened. Problem k
    owns rows [row_off[k], row_off[k] + n[k] + m[k]) of X: its n[k] sources,
    then its m[k] targets."""
    name: str
    X: np.ndarray            # total_rows x d float64 (fp32-representable)
    n: np.ndarray            # int32 per problem
    m: np.ndarray            # int32 per problem
    row_off: np.ndarray      # int64 per problem
    seeds: np.ndarray        # uint64 base seed per problem
    cost: int
    lam: float
    buckets: int
    kmeans_iters: int
    landmarks: int
    iters: int

    @property
    def count(self):
        return len(self.n)

    @property
    def d(self):
        return self.X.shape[1]

    def lsh_seed(self, k):
        return mix_seed(int(self.seeds[k]), 3)

    def landmark_seed(self, k):
        return mix_seed(int(self.seeds[k]), 4)

    def lsh_seeds(self):
        return mix_seed_array(self.seeds, 3)

    def landmark_seeds(self):
        return mix_seed_array(self.seeds, 4)

    def problem(self, k):
        o, n, m = int(self.row_off[k]), int(self.n[k]), int(self.m[k])
        return self.X[o:o + n], self.X[o + n:o + n + m]


def config4(scale: float = 1.0) -> Batch:
    """configs[4]: 4096 source/target pairs with node counts uniform in
    [20, 200], 64-d N(0,1) node embeddings; 8 heads per pair, each a seeded
    64->16 projection (entries N(0, 1/64)), rounded to fp32. Per (pair, head)
    problem: L2 cost, lambda = 0.1 (no lambda schedule: the config does not
    ask for one, recorded), LCN with 10 k-means landmarks, 1 x 8 k-means LSH,
    50 iterations. `scale` shrinks the number of pairs."""
    seed = 1004
    pairs = max(1, int(round(4096 * scale)))
    heads, d_in, d = 8, 64, 16
    rng = np.random.default_rng(seed)
    proj = (rng.standard_normal((heads, d_in, d), dtype=np.float32) * np.float32(0.125)).astype(np.float64)
    blocks, ns, ms = [], [], []
    for _ in range(pairs):
        n, m = int(rng.integers(20, 201)), int(rng.integers(20, 201))
        src = rng.standard_normal((n, d_in), dtype=np.float32).astype(np.float64)
        tgt = rng.standard_normal((m, d_in), dtype=np.float32).astype(np.float64)
        for h in range(heads):
            blocks.append((src @ proj[h]).astype(np.float32))
            blocks.append((tgt @ proj[h]).astype(np.float32))
            ns.append(n)
            ms.append(m)
    X = np.concatenate(blocks).astype(np.float64)
    n_arr, m_arr = np.array(ns, np.int32), np.array(ms, np.int32)
    row_off = np.concatenate([[0], np.cumsum(n_arr.astype(np.int64) + m_arr)[:-1]]).astype(np.int64)
    seeds = np.array([mix_seed(seed, 16 + k) for k in range(len(ns))], np.uint64)
    return Batch("c4_batched", X, n_arr, m_arr, row_off, seeds, EUCLIDEAN, 0.1, 8, 10, 10, 50)
