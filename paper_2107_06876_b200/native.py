"""Python host mirror of the reference's lcn:: solver API over the C-ABI.

Binds paper_2107_06876_b200/_build/liblcn_b200.so (include/lcn_b200.h) with
ctypes and exposes the reference's names and error types
(lsh.hpp, kmeans.hpp, nystrom.hpp, sparse_kernel.hpp, operator.hpp,
sinkhorn.hpp, error.hpp). There is no CPU fallback: if the library is missing
or no sm_100 device is present every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Optional

import numpy as np

LIB_PATH = os.environ.get("LCN_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build",
                                                         "liblcn_b200.so")  # LCN_LIB_PATH: a profiling build


# ---- error types (error.hpp:8-38) -------------------------------------------
class Error(RuntimeError):
    pass


class DimensionError(Error):
    pass


class InvalidArgument(Error):
    pass


class StabilizationError(Error):
    pass


class NegativeKernelError(Error):
    pass


class FactorizationError(Error):
    pass


class CudaError(Error):
    pass


_STATUS = {1: DimensionError, 2: InvalidArgument, 3: StabilizationError, 4: NegativeKernelError,
           5: FactorizationError, 6: Error, 100: CudaError, 101: CudaError}

# enums (include/lcn_b200.h)
EUCLIDEAN, NEGATIVE_DOT, COSINE_DERIVED, SQEUCLIDEAN = 0, 1, 2, 3
LANDMARK_KMEANS, LANDMARK_KMEANSPP = 0, 1
LSH_CROSS_POLYTOPE, LSH_KMEANS, LSH_HIERARCHICAL_KMEANS = 0, 1, 2  # LshScheme (lsh.hpp:13-17)
ABI_VERSION = 5  # include/lcn_b200.h LCN_B200_ABI_VERSION
KIND_DENSE, KIND_SPARSE, KIND_NYSTROM, KIND_LCN = 0, 1, 2, 3
_KIND_NAMES = {0: "dense", 1: "sparse", 2: "nystrom", 3: "lcn"}


class _LshConfig(C.Structure):
    _fields_ = [("bands", C.c_int), ("rows_per_band", C.c_int), ("buckets_per_fn", C.c_int),
                ("kmeans_iters", C.c_int), ("seed", C.c_uint64), ("scheme", C.c_int), ("branching", C.c_int)]


class _SinkOpts(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iters", C.c_int), ("check_support", C.c_int), ("want_plan", C.c_int)]


class _OpInfo(C.Structure):
    _fields_ = [("kind", C.c_int), ("n", C.c_size_t), ("m", C.c_size_t), ("l", C.c_size_t), ("d", C.c_size_t),
                ("bands", C.c_int), ("nnz", C.c_size_t), ("stored", C.c_size_t), ("lam", C.c_double),
                ("max_abs_delta", C.c_double), ("cond_estimate", C.c_double), ("store_fp64", C.c_int),
                ("streamed", C.c_size_t)]


class _ResInfo(C.Structure):
    _fields_ = [("distance", C.c_double), ("iters", C.c_int), ("converged", C.c_int),
                ("marginal_err_final", C.c_double), ("n_warnings", C.c_int), ("device_ms", C.c_double)]


_lib = None


class _ShardInfo(C.Structure):
    _fields_ = [(k, C.c_size_t) for k in ("n_own", "n_halo", "m_own", "m_halo", "exp_s", "exp_t", "max_exp_s",
                                          "max_exp_t")] + [("cost", C.c_double), ("band0_pairs", C.c_ulonglong),
                                                           ("groups", C.c_size_t)]


def _preload_nccl():
    """The library links libnccl.so.2. When PyTorch's bundled NCCL (newer than
    the system copy) is installed, load it first so both resolve to the same
    libnccl.so.2 whatever the import order (torch needs its own version's
    symbols; the NCCL calls here work on either)."""
    import sys
    for base in sys.path:
        cand = os.path.join(base, "nvidia", "nccl", "lib", "libnccl.so.2")
        if os.path.exists(cand):
            try:
                C.CDLL(cand, mode=C.RTLD_GLOBAL)
            except OSError:
                pass
            return


def library() -> C.CDLL:
    """Load the C-ABI library (fails loudly when it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C paper_2107_06876_b200)")
        _preload_nccl()
        lib = C.CDLL(LIB_PATH)
        P, SZ, D, I, U64 = C.c_void_p, C.c_size_t, C.c_double, C.c_int, C.c_uint64
        PP = C.POINTER(C.c_void_p)
        sig = {
            "lcn_abi_version": ([], I),
            "lcn_status_name": ([I], C.c_char_p),
            "lcn_ctx_create": ([I, I, PP], I),
            "lcn_ctx_destroy": ([P], I),
            "lcn_ctx_last_error": ([P], C.c_char_p),
            "lcn_ctx_set_stream": ([P, P], I),
            "lcn_ctx_set_profile": ([P, I], I),
            "lcn_ctx_tc_work": ([P, I, C.POINTER(C.c_ulonglong)], I),
            "lcn_sinkhorn_device": ([P, P, P, C.POINTER(_SinkOpts), PP], I),
            "lcn_result_phase_ms": ([P, P, C.POINTER(I)], I),
            "lcn_kmeans_pp_indices": ([P, P, SZ, SZ, SZ, U64, P, SZ, P, C.POINTER(SZ)], I),
            "lcn_assign_nearest": ([P, P, SZ, SZ, P, SZ, P], I),
            "lcn_lloyd": ([P, P, SZ, SZ, SZ, I, U64, P, P], I),
            "lcn_lsh_kmeans_buckets": ([P, P, SZ, P, SZ, SZ, C.POINTER(_LshConfig), P], I),
            "lcn_lsh_buckets": ([P, P, SZ, P, SZ, SZ, C.POINTER(_LshConfig), P], I),
            "lcn_cross_polytope_buckets": ([P, P, SZ, SZ, P, SZ, P], I),
            "lcn_batched_lcn": ([P, P, SZ, SZ, I, P, P, I, D, I, I, P, SZ, P, I, P, P, P], I),
            "lcn_op_sparse_lsh": ([P, P, SZ, P, SZ, SZ, I, D, C.POINTER(_LshConfig), PP], I),
            "lcn_op_sparse_buckets": ([P, P, SZ, P, SZ, SZ, I, D, P, P, I, U64, PP], I),
            "lcn_op_lcn_lsh": ([P, P, SZ, P, SZ, SZ, I, D, C.POINTER(_LshConfig), SZ, I, U64, PP], I),
            "lcn_op_lcn_buckets": ([P, P, SZ, P, SZ, SZ, I, D, P, P, I, U64, P, SZ, I, U64, PP], I),
            "lcn_op_create_device": ([P, P, SZ, P, SZ, SZ, I, D, C.POINTER(_LshConfig), SZ, I, U64, PP], I),
            "lcn_op_destroy": ([P], I),
            "lcn_op_get_info": ([P, C.POINTER(_OpInfo)], I),
            "lcn_op_export_csr": ([P, I, P, P, P], I),
            "lcn_op_export_factor": ([P, I, P], I),
            "lcn_op_log_matvec": ([P, P, I, P], I),
            "lcn_sinkhorn": ([P, P, P, C.POINTER(_SinkOpts), PP], I),
            "lcn_result_destroy": ([P], I),
            "lcn_result_get_info": ([P, C.POINTER(_ResInfo)], I),
            "lcn_result_copy": ([P, I, P, C.POINTER(SZ)], I),
            "lcn_distance_lcn": ([P, P, C.POINTER(D)], I),
            "lcn_result_warning": ([P, I], C.c_char_p),
            "lcn_nccl_unique_id": ([P], I),
            "lcn_op_dense": ([P, P, SZ, P, SZ, SZ, I, D, PP], I),
            "lcn_op_dense_device": ([P, P, SZ, P, SZ, SZ, I, D, PP], I),
            "lcn_op_export_dense": ([P, P], I),
            "lcn_grad_cost": ([P, P, I, P, C.POINTER(SZ), C.POINTER(I)], I),
            "lcn_multihead": ([P, P, SZ, P, SZ, SZ, I, D, I, P, P, C.POINTER(_SinkOpts), P, P, P, P, P], I),
            "lcn_ctx_set_comm": ([P, I, I, P], I),
            "lcn_loopback_create": ([I, PP], I),
            "lcn_ctx_set_loopback": ([P, P, I], I),
            "lcn_loopback_abort": ([P], I),
            "lcn_loopback_destroy": ([P], I),
            "lcn_shard_plan_create": ([P, SZ, P, SZ, I, P, SZ, I, PP], I),
            "lcn_shard_plan_rank_info": ([P, I, C.POINTER(_ShardInfo)], I),
            "lcn_shard_plan_rank_points": ([P, I, P, P], I),
            "lcn_shard_plan_rank_exchange": ([P, I, P, P, P, P, P, P], I),
            "lcn_shard_plan_last_error": ([], C.c_char_p),
            "lcn_shard_plan_destroy": ([P], I),
            "lcn_lsh_neighbor_pairs": ([P, P, SZ, P, SZ, SZ, C.POINTER(_LshConfig), PP], I),
            "lcn_pairs_info": ([P, C.POINTER(SZ), C.POINTER(SZ), C.POINTER(SZ)], I),
            "lcn_pairs_copy": ([P, P, P], I),
            "lcn_pairs_destroy": ([P], I),
            "lcn_build_sparse": ([P, P, SZ, P, SZ, SZ, P, P, SZ, I, D, P], I),
            "lcn_select_landmarks": ([P, P, SZ, P, SZ, SZ, SZ, I, U64, P], I),
            "lcn_build_factors": ([P, P, SZ, P, SZ, SZ, P, SZ, I, D, P, P, C.POINTER(D)], I),
            "lcn_build_correction": ([P, SZ, SZ, SZ, P, P, SZ, P, P, P, P, P, C.POINTER(D)], I),
            "lcn_op_from_dense": ([P, SZ, SZ, P, D, PP], I),
            "lcn_op_from_sparse": ([P, SZ, SZ, P, P, SZ, P, D, PP], I),
            "lcn_op_from_nystrom": ([P, SZ, SZ, SZ, P, P, D, PP], I),
            "lcn_op_from_lcn": ([P, SZ, SZ, SZ, P, P, D, P, P, SZ, P, P, D, PP], I),
            "lcn_op_set_bp": ([P, P, P], I),
        }
        for name, (args, res) in sig.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = res
        if lib.lcn_abi_version() != ABI_VERSION:
            raise ImportError(f"{LIB_PATH}: ABI {lib.lcn_abi_version()}, this mirror is ABI {ABI_VERSION} (rebuild)")
        _lib = lib
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None and a.shape != shape:
        raise DimensionError(f"expected shape {shape}, got {a.shape}")
    return a


class Context:
    """One device, one stream (lcn_ctx). store_fp64 selects fp64 storage of the
    iteration operands (API-compatibility precision) over fp32 (performance).
    exact_build (LCN_EXACT_BUILD) keeps the exact fp64 build tiles in fp32
    storage; otherwise fp32 storage builds K^sp, U, V and delta on the tensor
    cores (3xTF32)."""

    def __init__(self, device: int = 0, store_fp64: bool = False, exact_build: bool = False,
                 dense_recompute: bool = False):
        self.lib = library()
        h = C.c_void_p()
        flags = (1 if store_fp64 else 0) | (2 if exact_build else 0) | (4 if dense_recompute else 0)
        rc = self.lib.lcn_ctx_create(device, flags, C.byref(h))
        if rc != 0:
            raise _STATUS.get(rc, Error)(self.lib.lcn_ctx_last_error(None).decode())
        self.h = h
        self.device = device
        self.store_fp64 = store_fp64

    def check(self, rc: int):
        if rc != 0:
            raise _STATUS.get(rc, Error)(self.lib.lcn_ctx_last_error(self.h).decode())

    def set_stream(self, stream_handle: int | None):
        """Run on an external cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream)."""
        self.check(self.lib.lcn_ctx_set_stream(self.h, C.c_void_p(stream_handle) if stream_handle else None))

    def set_profile(self, on: bool):
        self.check(self.lib.lcn_ctx_set_profile(self.h, 1 if on else 0))

    def tc_work(self, reset: bool = False) -> int:
        """Point x 128-centroid tile products the tensor-core assignment
        filter evaluated since the last reset (lcn_ctx_tc_work)."""
        v = C.c_ulonglong(0)
        self.check(self.lib.lcn_ctx_tc_work(self.h, 1 if reset else 0, C.byref(v)))
        return int(v.value)

    def set_comm(self, world: int, rank: int, uid: bytes):
        """Join a sharded solve (lcn_ctx_set_comm): `uid` is rank 0's
        nccl_unique_id(), broadcast to every rank; collective over the ranks."""
        if len(uid) != 128:
            raise InvalidArgument("NCCL unique id must be 128 bytes")
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        self.check(self.lib.lcn_ctx_set_comm(self.h, int(world), int(rank), C.addressof(buf)))

    def set_loopback(self, group: "LoopbackGroup", rank: int):
        """Join an in-process loopback communicator (lcn_ctx_set_loopback):
        ranks as threads sharing a device, for testing the sharded path."""
        self.check(self.lib.lcn_ctx_set_loopback(self.h, group.h, int(rank)))
        self._group = group

    def close(self):
        # live operators keep a pointer to the context: its destruction waits
        # for the last one (finalizers run in any order in cyclic collection,
        # after weak references are cleared)
        if getattr(self, "h", None):
            if getattr(self, "_live", 0) > 0:
                self._close_pending = True
                return
            self.lib.lcn_ctx_destroy(self.h)
            self.h = None

    def _adopt(self, child):
        self._live = getattr(self, "_live", 0) + 1

    def _release(self):
        self._live -= 1
        if self._live == 0 and getattr(self, "_close_pending", False):
            self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LoopbackGroup:
    """lcn_loopback: `world` ranks as host threads of this process on one
    device; the all-gather is a host barrier plus device copies."""

    def __init__(self, world: int):
        self.lib = library()
        h = C.c_void_p()
        if self.lib.lcn_loopback_create(int(world), C.byref(h)) != 0:
            raise InvalidArgument(self.lib.lcn_ctx_last_error(None).decode())
        self.h = h
        self.world = world

    def abort(self):
        self.lib.lcn_loopback_abort(self.h)

    def __del__(self):
        try:
            if self.h:
                self.lib.lcn_loopback_destroy(self.h)
                self.h = None
        except Exception:
            pass


class ShardPlan:
    """The bucket-sharded partition the library builds (lcn_shard_plan_*;
    host only, no GPU): owned + halo points per rank and the exchange maps."""

    def __init__(self, ids_src, ids_tgt, ranges, l: int, world: int):
        self.lib = library()
        ids_src = np.ascontiguousarray(np.atleast_2d(ids_src), np.uint32)
        ids_tgt = np.ascontiguousarray(np.atleast_2d(ids_tgt), np.uint32)
        rng = np.ascontiguousarray(np.broadcast_to(np.asarray(ranges, np.uint32), (ids_src.shape[0],)))
        h = C.c_void_p()
        rc = self.lib.lcn_shard_plan_create(_p(ids_src), ids_src.shape[1], _p(ids_tgt), ids_tgt.shape[1],
                                            ids_src.shape[0], _p(rng), int(l), int(world), C.byref(h))
        if rc != 0:
            raise _STATUS.get(rc, Error)(self.lib.lcn_shard_plan_last_error().decode())
        self.h, self.world = h, world

    def info(self, rank: int) -> dict:
        inf = _ShardInfo()
        if self.lib.lcn_shard_plan_rank_info(self.h, rank, C.byref(inf)) != 0:
            raise InvalidArgument(self.lib.lcn_shard_plan_last_error().decode())
        return {k: getattr(inf, k) for k, _ in _ShardInfo._fields_}

    def points(self, rank: int):
        """(local -> global sources, local -> global targets): owned then halo."""
        i = self.info(rank)
        src = np.zeros(i["n_own"] + i["n_halo"], np.uint32)
        tgt = np.zeros(i["m_own"] + i["m_halo"], np.uint32)
        self.lib.lcn_shard_plan_rank_points(self.h, rank, _p(src), _p(tgt))
        return src, tgt

    def exchange(self, rank: int) -> dict:
        i = self.info(rank)
        out = {"exp_s": np.zeros(i["exp_s"], np.uint32), "exp_t": np.zeros(i["exp_t"], np.uint32)}
        for k, cnt in (("s", i["n_halo"]), ("t", i["m_halo"])):
            out[f"imp_{k}_rank"] = np.zeros(cnt, np.uint32)
            out[f"imp_{k}_slot"] = np.zeros(cnt, np.uint32)
        self.lib.lcn_shard_plan_rank_exchange(self.h, rank, _p(out["exp_s"]), _p(out["exp_t"]), _p(out["imp_s_rank"]),
                                              _p(out["imp_s_slot"]), _p(out["imp_t_rank"]), _p(out["imp_t_slot"]))
        return out

    def __del__(self):
        try:
            if self.h:
                self.lib.lcn_shard_plan_destroy(self.h)
                self.h = None
        except Exception:
            pass


# ---- staged build from host structs (runner.cpp:258-271) ---------------------
def _csr(row_ptr, col):
    return np.ascontiguousarray(row_ptr, np.uint32), np.ascontiguousarray(col, np.uint32)


def lsh_neighbor_pairs(ctx: "Context", p, q, cfg: "LshConfig"):
    """lsh_neighbor_pairs (lsh.cpp:245-283) -> (row_ptr, col) CSR."""
    p, q = _f64(p), _f64(q)
    h = C.c_void_p()
    c = cfg.c()
    ctx.check(ctx.lib.lcn_lsh_neighbor_pairs(ctx.h, _p(p), p.shape[0], _p(q), q.shape[0], p.shape[1], C.byref(c),
                                             C.byref(h)))
    try:
        nnz = C.c_size_t()
        ctx.lib.lcn_pairs_info(h, None, None, C.byref(nnz))
        rp = np.zeros(p.shape[0] + 1, np.uint32)
        col = np.zeros(nnz.value, np.uint32)
        ctx.lib.lcn_pairs_copy(h, _p(rp), _p(col))
    finally:
        ctx.lib.lcn_pairs_destroy(h)
    return rp, col


def build_sparse(ctx: "Context", p, q, row_ptr, col, cost, lam):
    """build_sparse (sparse_kernel.cpp:51-80): log K at the pattern."""
    p, q = _f64(p), _f64(q)
    rp, col = _csr(row_ptr, col)
    out = np.zeros(len(col))
    ctx.check(ctx.lib.lcn_build_sparse(ctx.h, _p(p), p.shape[0], _p(q), q.shape[0], p.shape[1], _p(rp), _p(col),
                                       len(col), cost, lam, _p(out)))
    return out


def select_landmarks(ctx: "Context", p, q, l: int, method=0, seed=0):
    p, q = _f64(p), _f64(q)
    out = np.zeros((l, p.shape[1]))
    ctx.check(ctx.lib.lcn_select_landmarks(ctx.h, _p(p), p.shape[0], _p(q), q.shape[0], p.shape[1], l, method, seed,
                                           _p(out)))
    return out


def build_factors(ctx: "Context", p, q, landmarks, cost, lam):
    """build_factors (nystrom.cpp:68-125) -> (U n x l, W l x m, cond)."""
    p, q, L = _f64(p), _f64(q), _f64(landmarks)
    l = L.shape[0]
    U = np.zeros((p.shape[0], l))
    W = np.zeros((l, q.shape[0]))
    cond = C.c_double()
    ctx.check(ctx.lib.lcn_build_factors(ctx.h, _p(p), p.shape[0], _p(q), q.shape[0], p.shape[1], _p(L), l, cost, lam,
                                        _p(U), _p(W), C.byref(cond)))
    return U, W, cond.value


def build_correction(ctx: "Context", row_ptr, col, log_sp, U, W):
    """build_correction (sparse_kernel.cpp:82-117) -> (delta, nys_vals, max |delta|)."""
    rp, col = _csr(row_ptr, col)
    U, W, ls = _f64(U), _f64(W), _f64(log_sp)
    delta = np.zeros(len(col))
    nys = np.zeros(len(col))
    mx = C.c_double()
    ctx.check(ctx.lib.lcn_build_correction(ctx.h, U.shape[0], W.shape[1], U.shape[1], _p(rp), _p(col), len(col),
                                           _p(ls), _p(U), _p(W), _p(delta), _p(nys), C.byref(mx)))
    return delta, nys, mx.value


@dataclasses.dataclass
class LshConfig:
    """LshConfig (lsh.hpp:22-30); scheme defaults to k-means like the reference."""
    bands: int = 1
    rows_per_band: int = 1
    buckets_per_fn: int = 2
    kmeans_iters: int = 10
    seed: int = 0
    scheme: int = LSH_KMEANS
    branching: int = 2

    def c(self):
        return _LshConfig(self.bands, self.rows_per_band, self.buckets_per_fn, self.kmeans_iters, self.seed,
                          self.scheme, self.branching)


@dataclasses.dataclass
class SinkhornOptions:
    """SinkhornOptions (sinkhorn.hpp:11-20)."""
    tol: float = -1.0
    max_iters: int = 500
    check_support: bool = True
    want_plan: bool = True

    def c(self):
        return _SinkOpts(self.tol, self.max_iters, int(self.check_support), int(self.want_plan))


# ---- k-means (kmeans.hpp:18-29) ----------------------------------------------
def kmeans_pp_indices(ctx: Context, points, k: int, rng: np.random.Generator | None = None, *, seed: int | None = None):
    """kmeans_pp_indices with a libstdc++ mt19937_64(seed) engine (the draws are
    taken by the C++ side of lloyd; here the caller passes the seed)."""
    import random  # noqa: F401  (documented: draws come from std::mt19937_64 in C)
    pts = _f64(points)
    n, d = pts.shape
    if seed is None:
        raise InvalidArgument("kmeans_pp_indices needs the engine seed")
    first, raw = _mt_draws(seed, n, max(k - 1, 0))
    out = np.zeros(k, np.uint32)
    used = C.c_size_t()
    rawa = np.ascontiguousarray(raw, np.uint64)
    ctx.check(ctx.lib.lcn_kmeans_pp_indices(ctx.h, _p(pts), n, d, k, first, _p(rawa), len(rawa), _p(out),
                                            C.byref(used)))
    return out


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (lcn_nccl_unique_id), to broadcast from rank 0."""
    lib = library()
    buf = (C.c_uint8 * 128)()
    st = lib.lcn_nccl_unique_id(C.addressof(buf))
    if st != 0:
        raise CudaError("lcn_nccl_unique_id failed")
    return bytes(buf)


def assign_nearest(ctx: Context, points, centroids):
    pts, ctr = _f64(points), _f64(centroids)
    out = np.zeros(pts.shape[0], np.uint32)
    ctx.check(ctx.lib.lcn_assign_nearest(ctx.h, _p(pts), pts.shape[0], pts.shape[1], _p(ctr), ctr.shape[0], _p(out)))
    return out


def lloyd(ctx: Context, points, k: int, iters: int, seed: int):
    """lloyd (kmeans.cpp:87-143) -> (centroids k x d, assign n)."""
    pts = _f64(points)
    n, d = pts.shape
    ctr = np.zeros((k, d))
    asg = np.zeros(n, np.uint32)
    ctx.check(ctx.lib.lcn_lloyd(ctx.h, _p(pts), n, d, k, iters, seed, _p(ctr), _p(asg)))
    return ctr, asg


def batched_lcn(ctx: Context, batch):
    """configs[4]: every problem of a configs.Batch in ragged launches (one
    CTA per problem). Returns (distances, statuses, iterations); a problem
    with a non-zero status (the reference's first error for it) has distance NaN."""
    X = _f64(batch.X)
    k = batch.count
    n = np.ascontiguousarray(batch.n, np.int32)
    m = np.ascontiguousarray(batch.m, np.int32)
    lsh = np.ascontiguousarray(batch.lsh_seeds(), np.uint64)
    lms = np.ascontiguousarray(batch.landmark_seeds(), np.uint64)
    dist = np.zeros(k)
    st = np.zeros(k, np.int32)
    it = np.zeros(k, np.int32)
    ctx.check(ctx.lib.lcn_batched_lcn(ctx.h, _p(X), X.shape[0], X.shape[1], k, _p(n), _p(m), batch.cost, batch.lam,
                                      batch.buckets, batch.kmeans_iters, _p(lsh), batch.landmarks, _p(lms),
                                      batch.iters, _p(dist), _p(st), _p(it)))
    return dist, st, it


def cross_polytope_buckets(ctx: Context, points, proj):
    """cross_polytope_bucket (lsh.cpp:55-71) per point; proj is d x half."""
    points = _f64(points)
    proj = np.ascontiguousarray(proj, np.float64)
    out = np.zeros(points.shape[0], np.uint32)
    ctx.check(ctx.lib.lcn_cross_polytope_buckets(ctx.h, _p(points), points.shape[0], points.shape[1], _p(proj),
                                                 proj.shape[1], _p(out)))
    return out


def lsh_buckets(ctx: Context, p, q, cfg: LshConfig):
    """Per-band composite bucket ids of lsh_neighbor_pairs (lsh.cpp:245-283) for cfg.scheme, p's points first."""
    return lsh_kmeans_buckets(ctx, p, q, cfg)


def lsh_kmeans_buckets(ctx: Context, p, q, cfg: LshConfig):
    """Per-band bucket ids on X_p ∪ X_q (lsh.cpp:245-283); honours cfg.scheme."""
    p, q = _f64(p), _f64(q)
    ids = np.zeros((cfg.bands, p.shape[0] + q.shape[0]), np.uint64)
    c = cfg.c()
    ctx.check(ctx.lib.lcn_lsh_kmeans_buckets(ctx.h, _p(p), p.shape[0], _p(q), q.shape[0], p.shape[1], C.byref(c),
                                             _p(ids)))
    return ids


def _mt_draws(seed: int, n: int, count: int):
    """first = uniform_int_distribution<size_t>(0, n-1)(mt19937_64(seed)) and the
    next `count` raw draws, computed by the library's own host code path."""
    # The C++ host side owns the engine; reproduce it with numpy's MT19937-64-free
    # implementation below (mt19937_64 is a fixed, standard algorithm).
    mt = _MT19937_64(seed)
    first = _lemire(mt, n)
    return first, [mt() for _ in range(count)]


class _MT19937_64:
    """std::mt19937_64 (a standard-specified engine)."""
    NN, MM = 312, 156
    MATRIX_A = 0xB5026F5AA96619E9
    UM, LM = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed: int):
        m = (1 << 64) - 1
        self.mt = [0] * self.NN
        self.mt[0] = seed & m
        for i in range(1, self.NN):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & m
        self.mti = self.NN

    def __call__(self) -> int:
        m = (1 << 64) - 1
        if self.mti >= self.NN:
            mt = self.mt
            for i in range(self.NN):
                x = (mt[i] & self.UM) | (mt[(i + 1) % self.NN] & self.LM)
                xa = x >> 1
                if x & 1:
                    xa ^= self.MATRIX_A
                mt[i] = mt[(i + self.MM) % self.NN] ^ xa
            self.mti = 0
        x = self.mt[self.mti]
        self.mti += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & m


def _lemire(mt, n: int) -> int:
    """libstdc++ uniform_int_distribution<size_t>(0, n-1): Lemire's nearly
    divisionless downscaling with a 128-bit product (uniform_int_dist.h)."""
    rng = n
    prod = mt() * rng
    low = prod & ((1 << 64) - 1)
    if low < rng:
        thr = ((1 << 64) - rng) % rng
        while low < thr:
            prod = mt() * rng
            low = prod & ((1 << 64) - 1)
    return prod >> 64


# ---- operators (operator.hpp:29-82) -----------------------------------------
class KernelOperator:
    """Device-resident kernel operator handle (lcn_op)."""

    def __init__(self, ctx: Context, h):
        self.ctx, self.h = ctx, h
        ctx._adopt(self)
        info = _OpInfo()
        ctx.check(ctx.lib.lcn_op_get_info(self.h, C.byref(info)))
        self.info = info

    # factories ---------------------------------------------------------------
    @classmethod
    def dense(cls, ctx, p, q, cost, lam):
        """build_cost -> build_kernel -> KernelOperator::dense (the configs[2] anchor)."""
        p, q = _f64(p), _f64(q)
        h = C.c_void_p()
        ctx.check(ctx.lib.lcn_op_dense(ctx.h, _p(p), p.shape[0], _p(q), q.shape[0], p.shape[1], cost, lam,
                                       C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def dense_device(cls, ctx, d_p: int, n: int, d_q: int, m: int, d: int, cost, lam):
        h = C.c_void_p()
        ctx.check(ctx.lib.lcn_op_dense_device(ctx.h, C.c_void_p(d_p), n, C.c_void_p(d_q), m, d, cost, lam,
                                              C.byref(h)))
        return cls(ctx, h)

    def export_dense(self):
        """DenseKernel::logk (n x m)."""
        out = np.zeros((self.n, self.m))
        self.ctx.check(self.ctx.lib.lcn_op_export_dense(self.h, _p(out)))
        return out

    @classmethod
    def sparse_lsh(cls, ctx, p, q, cost, lam, cfg: LshConfig):
        """lsh_neighbor_pairs -> build_sparse -> KernelOperator::sparse."""
        p, q = _f64(p), _f64(q)
        h = C.c_void_p()
        c = cfg.c()
        ctx.check(ctx.lib.lcn_op_sparse_lsh(ctx.h, _p(p), p.shape[0], _p(q), q.shape[0], p.shape[1], cost, lam,
                                            C.byref(c), C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def sparse_buckets(cls, ctx, p, q, cost, lam, ids_p, ids_q, range_=0):
        """neighbor_pairs(BandBuckets...) -> build_sparse -> KernelOperator::sparse."""
        p, q = _f64(p), _f64(q)
        ip = np.ascontiguousarray(np.atleast_2d(ids_p), np.uint64)
        iq = np.ascontiguousarray(np.atleast_2d(ids_q), np.uint64)
        h = C.c_void_p()
        ctx.check(ctx.lib.lcn_op_sparse_buckets(ctx.h, _p(p), p.shape[0], _p(q), q.shape[0], p.shape[1], cost, lam,
                                                _p(ip), _p(iq), ip.shape[0], range_, C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def lcn_lsh(cls, ctx, p, q, cost, lam, cfg: LshConfig, l: int, method=LANDMARK_KMEANS, landmark_seed=0):
        """lsh_neighbor_pairs + select_landmarks + build_factors + build_correction -> KernelOperator::lcn."""
        p, q = _f64(p), _f64(q)
        h = C.c_void_p()
        c = cfg.c()
        ctx.check(ctx.lib.lcn_op_lcn_lsh(ctx.h, _p(p), p.shape[0], _p(q), q.shape[0], p.shape[1], cost, lam,
                                         C.byref(c), l, method, landmark_seed, C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def lcn_buckets(cls, ctx, p, q, cost, lam, ids_p, ids_q, l=0, method=LANDMARK_KMEANS, landmark_seed=0,
                    landmarks=None, range_=0):
        """External bucket ids (+ optional explicit landmarks); no bands -> Nystrom operator."""
        p, q = _f64(p), _f64(q)
        if ids_p is None:
            ip = iq = np.zeros((0, 1), np.uint64)
            bands = 0
        else:
            ip = np.ascontiguousarray(np.atleast_2d(ids_p), np.uint64)
            iq = np.ascontiguousarray(np.atleast_2d(ids_q), np.uint64)
            bands = ip.shape[0]
        lm = None if landmarks is None else _f64(landmarks)
        if lm is not None:
            l = lm.shape[0]
        h = C.c_void_p()
        ctx.check(ctx.lib.lcn_op_lcn_buckets(ctx.h, _p(p), p.shape[0], _p(q), q.shape[0], p.shape[1], cost, lam,
                                             _p(ip), _p(iq), bands, range_, _p(lm), l, method, landmark_seed,
                                             C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def from_dense_logk(cls, ctx, logk, lam):
        """KernelOperator::dense(DenseKernel) from a host n x m log K."""
        lk = _f64(logk)
        h = C.c_void_p()
        ctx.check(ctx.lib.lcn_op_from_dense(ctx.h, lk.shape[0], lk.shape[1], _p(lk), lam, C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def from_sparse(cls, ctx, n, m, row_ptr, col, logvals, lam):
        """KernelOperator::sparse(SparseKernel, lambda), any CSR pattern."""
        rp, col = _csr(row_ptr, col)
        lv = _f64(logvals)
        h = C.c_void_p()
        ctx.check(ctx.lib.lcn_op_from_sparse(ctx.h, n, m, _p(rp), _p(col), len(col), _p(lv), lam, C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def from_nystrom(cls, ctx, U, W, lam):
        """KernelOperator::nystrom(NystromFactors)."""
        U, W = _f64(U), _f64(W)
        h = C.c_void_p()
        ctx.check(ctx.lib.lcn_op_from_nystrom(ctx.h, U.shape[0], W.shape[1], U.shape[1], _p(U), _p(W), lam,
                                              C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def from_lcn(cls, ctx, U, W, lam, row_ptr, col, delta, log_sp, max_abs_delta=0.0):
        """KernelOperator::lcn(NystromFactors, LcnCorrection), any CSR pattern."""
        U, W = _f64(U), _f64(W)
        rp, col = _csr(row_ptr, col)
        dl, ls = _f64(delta), _f64(log_sp)
        h = C.c_void_p()
        ctx.check(ctx.lib.lcn_op_from_lcn(ctx.h, U.shape[0], W.shape[1], U.shape[1], _p(U), _p(W), lam, _p(rp), _p(col),
                                          len(col), _p(dl), _p(ls), max_abs_delta, C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def from_device(cls, ctx, d_p: int, n: int, d_q: int, m: int, d: int, cost, lam, cfg: LshConfig, l=0,
                    method=LANDMARK_KMEANS, landmark_seed=0):
        """Device-resident fp32 points (raw device pointers, e.g. torch .data_ptr())."""
        h = C.c_void_p()
        c = cfg.c()
        ctx.check(ctx.lib.lcn_op_create_device(ctx.h, C.c_void_p(d_p), n, C.c_void_p(d_q), m, d, cost, lam,
                                               C.byref(c), l, method, landmark_seed, C.byref(h)))
        return cls(ctx, h)

    # accessors ---------------------------------------------------------------
    def kind(self):
        return _KIND_NAMES[self.info.kind]

    name = kind
    n = property(lambda s: s.info.n)
    m = property(lambda s: s.info.m)
    l = property(lambda s: s.info.l)
    nnz = property(lambda s: s.info.nnz)
    stored = property(lambda s: s.info.stored)
    streamed = property(lambda s: s.info.streamed)
    lam = property(lambda s: s.info.lam)
    max_abs_delta = property(lambda s: s.info.max_abs_delta)
    cond_estimate = property(lambda s: s.info.cond_estimate)

    def export_csr(self, which: int = 0):
        """(row_ptr, col, vals): which 0 log K^sp, 1 delta, 2 log_sp, 3 nys_vals."""
        rp = np.zeros(self.n + 1, np.uint32)
        col = np.zeros(max(self.nnz, 1), np.uint32)
        val = np.zeros(max(self.nnz, 1))
        self.ctx.check(self.ctx.lib.lcn_op_export_csr(self.h, which, _p(rp), _p(col), _p(val)))
        return rp, col[: self.nnz], val[: self.nnz]

    def factor(self, which: int):
        """0 U (n x l), 1 W (l x m), 2 landmarks (l x d)."""
        shape = {0: (self.n, self.l), 1: (self.l, self.m), 2: (self.l, self.info.d)}[which]
        out = np.zeros(shape)
        self.ctx.check(self.ctx.lib.lcn_op_export_factor(self.h, which, _p(out)))
        return out

    def with_bp(self, cost_p, cost_q):
        """KernelOperator::with_bp(BpExtension::from_costs(cost_p, cost_q, lambda))
        (operator.cpp:33-43, 103-115), applied to this operator in place."""
        cp, cq = _f64(cost_p, (self.n,)), _f64(cost_q, (self.m,))
        if not (self.lam > 0.0):
            raise InvalidArgument("BpExtension: lambda must be positive")
        dp, dq = np.exp(-cp / self.lam), np.exp(-cq / self.lam)
        self.ctx.check(self.ctx.lib.lcn_op_set_bp(self.h, _p(dp), _p(dq)))
        return self

    def log_matvec(self, log_t):
        v = _f64(log_t)
        if v.shape != (self.m,):
            raise DimensionError("log_matvec: vector length mismatch")
        out = np.zeros(self.n)
        self.ctx.check(self.ctx.lib.lcn_op_log_matvec(self.h, _p(v), 0, _p(out)))
        return out

    def log_matvec_t(self, log_s):
        v = _f64(log_s)
        if v.shape != (self.n,):
            raise DimensionError("log_matvec_t: vector length mismatch")
        out = np.zeros(self.m)
        self.ctx.check(self.ctx.lib.lcn_op_log_matvec(self.h, _p(v), 1, _p(out)))
        return out

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.lcn_op_destroy(self.h)
            self.h = None
            self.ctx._release()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class SinkhornResult:
    def __init__(self, op: KernelOperator, h):
        self.op, self.h = op, h
        info = _ResInfo()
        op.ctx.check(op.ctx.lib.lcn_result_get_info(h, C.byref(info)))
        self.distance = info.distance
        self.iters = info.iters
        self.converged = bool(info.converged)
        self.marginal_err_final = info.marginal_err_final
        self.device_ms = info.device_ms
        self.warnings = [op.ctx.lib.lcn_result_warning(h, i).decode() for i in range(info.n_warnings)]

    def phase_ms(self):
        """Profiling: summed ms of (col bands, col finalize+reduce, row bands, row
        finalize+reduce+end) over the iterations, and the iteration count."""
        out = np.zeros(4)
        it = C.c_int()
        self.op.ctx.check(self.op.ctx.lib.lcn_result_phase_ms(self.h, _p(out), C.byref(it)))
        return out, it.value

    def _vec(self, which):
        lib = self.op.ctx.lib
        n = C.c_size_t()
        lib.lcn_result_copy(self.h, which, None, C.byref(n))
        out = np.zeros(n.value)
        if n.value:
            lib.lcn_result_copy(self.h, which, _p(out), C.byref(n))
        return out

    log_s = property(lambda s: s._vec(0))
    log_t = property(lambda s: s._vec(1))
    row_marginal = property(lambda s: s._vec(2))
    marginal_err = property(lambda s: s._vec(3))
    sparse_vals = property(lambda s: s._vec(4))
    sp_vals = property(lambda s: s._vec(5))
    sp_nys_vals = property(lambda s: s._vec(6))
    del_p_mass = property(lambda s: s._vec(7))
    del_q_mass = property(lambda s: s._vec(8))
    eps_mass = property(lambda s: float(s._vec(9)[0]))

    def close(self):
        if getattr(self, "h", None):
            self.op.ctx.lib.lcn_result_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def sinkhorn(op: KernelOperator, p, q, opts: SinkhornOptions = SinkhornOptions()) -> SinkhornResult:
    """sinkhorn (sinkhorn.cpp:104-188)."""
    p = _f64(p)
    q = _f64(q)
    if p.shape != (op.n,) or q.shape != (op.m,):
        raise DimensionError("sinkhorn: marginal length does not match operator shape")
    o = _SinkOpts(opts.tol, opts.max_iters, int(opts.check_support), int(opts.want_plan))
    h = C.c_void_p()
    op.ctx.check(op.ctx.lib.lcn_sinkhorn(op.h, _p(p), _p(q), C.byref(o), C.byref(h)))
    return SinkhornResult(op, h)


def sinkhorn_device(op: KernelOperator, d_p: int, d_q: int, opts: SinkhornOptions = SinkhornOptions()):
    """sinkhorn on device-resident fp64 marginals (raw device pointers); no plan."""
    o = _SinkOpts(opts.tol, opts.max_iters, int(opts.check_support), 0)
    h = C.c_void_p()
    op.ctx.check(op.ctx.lib.lcn_sinkhorn_device(op.h, C.c_void_p(d_p), C.c_void_p(d_q), C.byref(o), C.byref(h)))
    return SinkhornResult(op, h)


def multihead(ctx: Context, p, q, cost, lam: float, heads: int, pm, qm,
              opts: SinkhornOptions = SinkhornOptions()):
    """multihead_lambdas + multihead (sinkhorn.cpp:322-353): one dense solve per
    lambda_k = 2^(k - heads/2) lambda; a failing head is reported, not raised.
    Returns a list of dicts {lambda, distance, iters, converged, status, error}."""
    p, q, pm, qm = _f64(p), _f64(q), _f64(pm), _f64(qm)
    lam_o, dist_o = np.zeros(heads), np.zeros(heads)
    it_o, cv_o, st_o = np.zeros(heads, np.int32), np.zeros(heads, np.int32), np.zeros(heads, np.int32)
    so = opts.c()
    ctx.check(ctx.lib.lcn_multihead(ctx.h, _p(p), p.shape[0], _p(q), q.shape[0], p.shape[1], cost, lam, heads,
                                    _p(pm), _p(qm), C.byref(so), _p(lam_o), _p(dist_o), _p(it_o), _p(cv_o),
                                    _p(st_o)))
    err = ctx.lib.lcn_ctx_last_error(ctx.h)
    return [{"lambda": float(lam_o[k]), "distance": float(dist_o[k]), "iters": int(it_o[k]),
             "converged": bool(cv_o[k]), "status": int(st_o[k]),
             "error": (err.decode() if err else "") if st_o[k] else ""} for k in range(heads)]


def grad_cost(res: SinkhornResult, op: KernelOperator, which: int):
    """grad_cost (sinkhorn.cpp:263-320): which 0 d/dC (dense n x m / sparse CSR
    order), 1 d/dU (n x l), 2 d/dW (l x m), 3 d/dlog K^sp, 4 d/dlog K^sp_Nys.
    Returns (array, stale)."""
    lib = op.ctx.lib
    n = C.c_size_t()
    st = C.c_int()
    op.ctx.check(lib.lcn_grad_cost(res.h, op.h, which, None, C.byref(n), C.byref(st)))
    out = np.zeros(n.value)
    op.ctx.check(lib.lcn_grad_cost(res.h, op.h, which, _p(out), C.byref(n), C.byref(st)))
    return out, bool(st.value)


def distance_lcn(res: SinkhornResult, op: KernelOperator) -> float:
    """distance_lcn (sinkhorn.cpp:222-261)."""
    out = C.c_double()
    op.ctx.check(op.ctx.lib.lcn_distance_lcn(res.h, op.h, C.byref(out)))
    return out.value


# ---- data formats and generators either side of the path (host only) -------
def _io_check(lib, rc: int):
    if rc != 0:
        raise _STATUS.get(rc, Error)(lib.lcn_io_last_error().decode())


def _io_lib():
    lib = library()
    if not getattr(lib, "_io_sigs", False):
        P, SZ, U64, I = C.c_void_p, C.c_size_t, C.c_uint64, C.c_int
        for name, args in {"lcn_points_read": [C.c_char_p, P, C.POINTER(SZ), C.POINTER(SZ)],
                           "lcn_points_write": [C.c_char_p, P, SZ, SZ, I],
                           "lcn_sample_uniform_ball": [SZ, SZ, U64, P],
                           "lcn_sample_clustered": [SZ, SZ, SZ, C.c_double, C.c_double, U64, P, P, P]}.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = I
        lib.lcn_io_last_error.argtypes = []
        lib.lcn_io_last_error.restype = C.c_char_p
        lib._io_sigs = True
    return lib


def read_points_file(path: str) -> np.ndarray:
    """read_points_file (io.cpp:105-116): LCNPTS1 binary or text, validated."""
    lib = _io_lib()
    n, d = C.c_size_t(0), C.c_size_t(0)
    _io_check(lib, lib.lcn_points_read(os.fsencode(path), None, C.byref(n), C.byref(d)))
    out = np.empty((n.value, d.value))
    _io_check(lib, lib.lcn_points_read(os.fsencode(path), _p(out), C.byref(n), C.byref(d)))
    return out


def write_points_file(path: str, points, binary: bool = True) -> None:
    """write_points_file (io.cpp:118-126)."""
    x = _f64(points)
    if x.ndim != 2:
        raise DimensionError("write_points_file: points must be n x d")
    lib = _io_lib()
    _io_check(lib, lib.lcn_points_write(os.fsencode(path), _p(x), x.shape[0], x.shape[1], int(bool(binary))))


def sample_uniform_ball(n: int, d: int, seed: int) -> np.ndarray:
    """sample_uniform_ball (generators.cpp:26-40), the reference's draws."""
    lib = _io_lib()
    out = np.empty((n, d)) if n and d else np.empty((0, 0))
    _io_check(lib, lib.lcn_sample_uniform_ball(n, d, seed, _p(out) if out.size else None))
    return out


def sample_clustered(n: int, d: int, c: int, D: float, r: float, seed: int):
    """sample_clustered (generators.cpp:42-106): (p, q, centers)."""
    lib = _io_lib()
    ok = n and d and c
    p, q = (np.empty((n, d)), np.empty((n, d))) if ok else (np.empty((0, 0)), np.empty((0, 0)))
    ctr = np.empty((c, d)) if ok else np.empty((0, 0))
    _io_check(lib, lib.lcn_sample_clustered(n, d, c, D, r, seed, _p(p) if ok else None, _p(q) if ok else None,
                                            _p(ctr) if ok else None))
    return p, q, ctr
