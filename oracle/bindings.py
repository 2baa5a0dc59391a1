"""ORACLE TEST INFRASTRUCTURE: ctypes bindings for the CPU checkers.

Two backends share one Python surface:
  * ``RefLib``    — oracle/_ref/libref_lcn.so, the reference's own C++ sources
                    compiled unmodified (oracle/Makefile ``make ref``);
  * ``OracleLib`` — oracle/_build/liblcn_oracle.so, the C restatement
                    (oracle/lcn_oracle.c).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module, and only as the checker.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libref_lcn.so")
ORACLE_SO = os.path.join(HERE, "_build", "liblcn_oracle.so")

_P = C.c_void_p
_SZ = C.c_size_t
_U64 = C.c_uint64
_D = C.c_double
_I = C.c_int
_PP = C.POINTER(C.c_void_p)

ERRORS = {1: "DimensionError", 2: "InvalidArgument", 3: "StabilizationError", 4: "NegativeKernelError",
          5: "FactorizationError", 6: "Error", 9: "Error"}


class LcnError(RuntimeError):
    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind
        self.msg = msg


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class _Lib:
    prefix = ""

    def __init__(self, path):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.lib = C.CDLL(path)
        self.path = path

    def fn(self, name, *argtypes, restype=C.c_int):
        f = getattr(self.lib, self.prefix + name)
        f.argtypes = list(argtypes)
        f.restype = restype
        return f

    def check(self, rc):
        if rc != 0:
            err = self.fn("last_error", restype=C.c_char_p)()
            raise LcnError(ERRORS.get(rc, "Error"), err.decode())


class CheckerLib(_Lib):
    """Common API exported with a per-backend prefix (ref_ / orc_)."""

    def kmeans_pp(self, pts, k, seed):
        pts = _f64(pts)
        out = np.zeros(k, np.uint32)
        self.check(self.fn("kmeans_pp", _P, _SZ, _SZ, _SZ, _U64, _P)(_ptr(pts), pts.shape[0], pts.shape[1], k,
                                                                       seed, _ptr(out)))
        return out

    def assign_nearest(self, pts, ctr):
        pts, ctr = _f64(pts), _f64(ctr)
        out = np.zeros(pts.shape[0], np.uint32)
        self.check(self.fn("assign_nearest", _P, _SZ, _SZ, _P, _SZ, _P)(_ptr(pts), pts.shape[0], pts.shape[1],
                                                                          _ptr(ctr), ctr.shape[0], _ptr(out)))
        return out

    def lloyd(self, pts, k, iters, seed):
        pts = _f64(pts)
        n, d = pts.shape
        ctr = np.zeros((k, d))
        asg = np.zeros(n, np.uint32)
        self.check(self.fn("lloyd", _P, _SZ, _SZ, _SZ, _I, _U64, _P, _P)(_ptr(pts), n, d, k, iters, seed,
                                                                           _ptr(ctr), _ptr(asg)))
        return ctr, asg

    def lsh_buckets(self, p, q, bands, buckets, iters, seed):
        p, q = _f64(p), _f64(q)
        ids = np.zeros((bands, p.shape[0] + q.shape[0]), np.uint64)
        self.check(self.fn("lsh_kmeans_buckets", _P, _SZ, _P, _SZ, _SZ, _I, _I, _I, _U64, _P)(
            _ptr(p), p.shape[0], _ptr(q), q.shape[0], p.shape[1], bands, buckets, iters, seed, _ptr(ids)))
        return ids

    def lcn_problem(self, p, q, kind, lam, buckets, kmeans_iters, lsh_seed, l, lm_seed, iters):
        """configs[4] unit: one small LCN solve end to end; returns the distance."""
        p, q = _f64(p), _f64(q)
        out = C.c_double()
        self.check(self.fn("lcn_problem", _P, _SZ, _P, _SZ, _SZ, _I, _D, _I, _I, _U64, _SZ, _U64, _I,
                           C.POINTER(C.c_double))(_ptr(p), p.shape[0], _ptr(q), q.shape[0], p.shape[1], kind, lam,
                                                  buckets, kmeans_iters, lsh_seed, l, lm_seed, iters, C.byref(out)))
        return out.value

    def lsh_buckets_cfg(self, p, q, scheme, bands=1, rows=1, buckets=2, iters=10, branching=2, seed=0):
        """Per-band composite ids (lsh.cpp:245-283) for any LshScheme value, p first."""
        p, q = _f64(p), _f64(q)
        ids = np.zeros((bands, p.shape[0] + q.shape[0]), np.uint64)
        self.check(self.fn("lsh_buckets", _P, _SZ, _P, _SZ, _SZ, _I, _I, _I, _I, _I, _I, _U64, _P)(
            _ptr(p), p.shape[0], _ptr(q), q.shape[0], p.shape[1], scheme, bands, rows, buckets, iters, branching,
            seed, _ptr(ids)))
        return ids

    def cross_polytope_bucket(self, x, proj):
        x = _f64(x)
        proj = _f64(proj)
        out = np.zeros(x.shape[0], np.uint32)
        self.check(self.fn("cross_polytope_bucket", _P, _SZ, _SZ, _P, _SZ, _P)(
            _ptr(x), x.shape[0], x.shape[1], _ptr(proj), proj.shape[1], _ptr(out)))
        return out

    def normal_draws(self, seed, count):
        out = np.zeros(count)
        self.check(self.fn("normal_draws", _U64, _SZ, _P)(seed, count, _ptr(out)))
        return out

    def _pairs_out(self, h):
        nnz = self.fn("pairs_nnz", _P, restype=_SZ)(h)
        rows = np.zeros(nnz, np.uint32)
        cols = np.zeros(nnz, np.uint32)
        if nnz:
            self.fn("pairs_copy", _P, _P, _P, restype=None)(h, _ptr(rows), _ptr(cols))
        return rows, cols

    def lsh_pairs(self, p, q, bands, buckets, iters, seed):
        """Returns a Pairs handle (rows, cols sorted row-major, unique)."""
        p, q = _f64(p), _f64(q)
        h = _P()
        self.check(self.fn("lsh_pairs", _P, _SZ, _P, _SZ, _SZ, _I, _I, _I, _U64, _PP)(
            _ptr(p), p.shape[0], _ptr(q), q.shape[0], p.shape[1], bands, buckets, iters, seed, C.byref(h)))
        return Pairs(self, h, p.shape[0], q.shape[0])

    def pairs_from_buckets(self, ids_p, ids_q, range_):
        ids_p = np.ascontiguousarray(ids_p, np.uint64)
        ids_q = np.ascontiguousarray(ids_q, np.uint64)
        h = _P()
        self.check(self.fn("pairs_from_buckets", _P, _SZ, _P, _SZ, _I, _U64, _PP)(
            _ptr(ids_p), ids_p.shape[1], _ptr(ids_q), ids_q.shape[1], ids_p.shape[0], range_, C.byref(h)))
        return Pairs(self, h, ids_p.shape[1], ids_q.shape[1])

    def pairs_from_arrays(self, n, m, rows, cols):
        rows = np.ascontiguousarray(rows, np.uint32)
        cols = np.ascontiguousarray(cols, np.uint32)
        h = _P()
        self.check(self.fn("pairs_from_arrays", _SZ, _SZ, _P, _P, _SZ, _PP)(n, m, _ptr(rows), _ptr(cols),
                                                                            len(rows), C.byref(h)))
        return Pairs(self, h, n, m)

    def op_sparse(self, p, q, kind, lam, pairs):
        p, q = _f64(p), _f64(q)
        h = _P()
        self.check(self.fn("op_sparse", _P, _SZ, _P, _SZ, _SZ, _I, _D, _P, _PP)(
            _ptr(p), p.shape[0], _ptr(q), q.shape[0], p.shape[1], kind, lam, pairs.h, C.byref(h)))
        return Op(self, h, p.shape[0], q.shape[0], "sparse")

    def op_lcn(self, p, q, kind, lam, pairs, l, method=0, lm_seed=0, landmarks=None, nystrom_only=False,
               phases=None):
        """phases (optional list) receives [select_landmarks, build_factors, build_sparse,
        build_correction] milliseconds (only the reference backend measures them)."""
        p, q = _f64(p), _f64(q)
        lm = _f64(landmarks) if landmarks is not None else None
        if lm is not None:
            l = lm.shape[0]
        h = _P()
        ph = np.zeros(4)
        self.check(self.fn("op_lcn", _P, _SZ, _P, _SZ, _SZ, _I, _D, _P, _SZ, _I, _U64, _P, _I, _PP, _P)(
            _ptr(p), p.shape[0], _ptr(q), q.shape[0], p.shape[1], kind, lam, pairs.h if pairs else None, l,
            method, lm_seed, _ptr(lm), int(nystrom_only), C.byref(h), _ptr(ph)))
        if phases is not None:
            phases[:] = list(ph)
        return Op(self, h, p.shape[0], q.shape[0], "nystrom" if nystrom_only else "lcn", l)

    def op_dense(self, p, q, kind, lam):
        p, q = _f64(p), _f64(q)
        h = _P()
        self.check(self.fn("op_dense", _P, _SZ, _P, _SZ, _SZ, _I, _D, _PP)(
            _ptr(p), p.shape[0], _ptr(q), q.shape[0], p.shape[1], kind, lam, C.byref(h)))
        return Op(self, h, p.shape[0], q.shape[0], "dense")

    def multihead(self, p, q, kind, lam, heads, pm, qm, tol=-1.0, max_iters=500):
        p, q, pm, qm = _f64(p), _f64(q), _f64(pm), _f64(qm)
        lam_o, dist_o = np.zeros(heads), np.zeros(heads)
        it_o, cv_o, er_o = np.zeros(heads, np.int32), np.zeros(heads, np.int32), np.zeros(heads, np.int32)
        self.check(self.fn("multihead", _P, _SZ, _P, _SZ, _SZ, _I, _D, _I, _P, _P, _D, _I, _P, _P, _P, _P, _P)(
            _ptr(p), p.shape[0], _ptr(q), q.shape[0], p.shape[1], kind, lam, heads, _ptr(pm), _ptr(qm), tol,
            max_iters, _ptr(lam_o), _ptr(dist_o), _ptr(it_o), _ptr(cv_o), _ptr(er_o)))
        return lam_o, dist_o, it_o, cv_o, er_o

    def dense_reference(self, cost, pm, qm, lam, tol, max_iters):
        cost, pm, qm = _f64(cost), _f64(pm), _f64(qm)
        n, m = cost.shape
        plan = np.zeros((n, m))
        dist = C.c_double()
        iters = C.c_int()
        self.check(self.fn("dense_reference", _P, _SZ, _SZ, _P, _P, _D, _D, _I, _P, C.POINTER(C.c_double),
                           C.POINTER(C.c_int))(_ptr(cost), n, m, _ptr(pm), _ptr(qm), lam, tol, max_iters,
                                               _ptr(plan), C.byref(dist), C.byref(iters)))
        return plan, dist.value, iters.value


class Pairs:
    def __init__(self, lib, h, n, m):
        self.lib, self.h, self.n, self.m = lib, h, n, m

    def arrays(self):
        return self.lib._pairs_out(self.h)

    def __del__(self):
        try:
            self.lib.fn("pairs_free", _P, restype=None)(self.h)
        except Exception:
            pass


class Op:
    def __init__(self, lib, h, n, m, kind, l=0):
        self.lib, self.h, self.n, self.m, self.kind, self.l = lib, h, n, m, kind, l

    def __del__(self):
        try:
            self.lib.fn("op_free", _P, restype=None)(self.h)
        except Exception:
            pass

    @property
    def nnz(self):
        return self.lib.fn("op_nnz", _P, restype=_SZ)(self.h)

    def scalar(self, which):
        return self.lib.fn("op_scalar", _P, _I, restype=_D)(self.h, which)

    def csr(self, which=0):
        nnz = self.nnz
        rp = np.zeros(self.n + 1, np.uint32)
        col = np.zeros(nnz, np.uint32)
        val = np.zeros(nnz)
        self.lib.check(self.lib.fn("op_copy", _P, _I, _P, _P, _P)(self.h, which, _ptr(rp), _ptr(col), _ptr(val)))
        return rp, col, val

    def dense_logk(self):
        out = np.zeros((self.n, self.m))
        self.lib.check(self.lib.fn("op_copy", _P, _I, _P, _P, _P)(self.h, 7, None, None, _ptr(out)))
        return out

    def dense_factor(self, which):
        shape = {2: (self.n, self.l), 3: (self.l, self.m)}[which]
        out = np.zeros(shape)
        self.lib.check(self.lib.fn("op_copy", _P, _I, _P, _P, _P)(self.h, which, None, None, _ptr(out)))
        return out

    def with_bp(self, cost_p, cost_q, lam):
        """KernelOperator::with_bp(BpExtension::from_costs(...)) in place."""
        cp, cq = _f64(cost_p), _f64(cost_q)
        self.lib.check(self.lib.fn("op_with_bp", _P, _P, _SZ, _P, _SZ, C.c_double)(self.h, _ptr(cp), len(cp), _ptr(cq),
                                                                                    len(cq), lam))
        return self

    def log_matvec(self, v, transposed=False):
        v = _f64(v)
        out = np.zeros(self.m if transposed else self.n)
        self.lib.check(self.lib.fn("op_log_matvec", _P, _P, _SZ, _I, _P)(self.h, _ptr(v), len(v), int(transposed),
                                                                           _ptr(out)))
        return out

    def sinkhorn(self, pm, qm, tol=-1.0, max_iters=500, check_support=True, want_plan=True):
        pm, qm = _f64(pm), _f64(qm)
        h = _P()
        self.lib.check(self.lib.fn("sinkhorn", _P, _P, _SZ, _P, _SZ, _D, _I, _I, _I, _PP)(
            self.h, _ptr(pm), len(pm), _ptr(qm), len(qm), tol, max_iters, int(check_support), int(want_plan),
            C.byref(h)))
        return Result(self.lib, h, self)


class Result:
    def __init__(self, lib, h, op):
        self.lib, self.h, self.op = lib, h, op

    def __del__(self):
        try:
            self.lib.fn("result_free", _P, restype=None)(self.h)
        except Exception:
            pass

    def _s(self, which):
        return self.lib.fn("result_scalar", _P, _I, restype=_D)(self.h, which)

    def _v(self, which):
        f = self.lib.fn("result_copy", _P, _I, _P, restype=_SZ)
        n = f(self.h, which, None)
        out = np.zeros(n)
        if n:
            f(self.h, which, _ptr(out))
        return out

    distance = property(lambda s: s._s(0))
    iters = property(lambda s: int(s._s(1)))
    converged = property(lambda s: bool(s._s(2)))
    marginal_err_final = property(lambda s: s._s(3))
    n_warnings = property(lambda s: int(s._s(4)))
    log_s = property(lambda s: s._v(0))
    log_t = property(lambda s: s._v(1))
    row_marginal = property(lambda s: s._v(2))
    marginal_err = property(lambda s: s._v(3))
    sparse_vals = property(lambda s: s._v(4))
    sp_vals = property(lambda s: s._v(5))
    sp_nys_vals = property(lambda s: s._v(6))
    dense_plan = property(lambda s: s._v(9))
    del_p_mass = property(lambda s: s._v(10))
    del_q_mass = property(lambda s: s._v(11))
    eps_mass = property(lambda s: s._s(6))

    def grad_cost(self, which):
        f = self.lib.fn("grad_cost", _P, _P, _I, _P, _P, restype=_SZ)
        stale = C.c_int()
        n = f(self.op.h, self.h, which, None, C.byref(stale))
        out = np.zeros(n)
        if n:
            f(self.op.h, self.h, which, _ptr(out), C.byref(stale))
        return out, bool(stale.value)

    def distance_lcn(self):
        out = C.c_double()
        self.lib.check(self.lib.fn("distance_lcn", _P, _P, C.POINTER(C.c_double))(self.h, self.op.h, C.byref(out)))
        return out.value


class RefLib(CheckerLib):
    prefix = "ref_"

    def __init__(self, path=REF_SO):
        super().__init__(path)

    def points_read(self, path):
        """read_points_file (io.cpp:105-116)."""
        n, d = _SZ(0), _SZ(0)
        f = self.fn("points_read", C.c_char_p, _P, C.POINTER(_SZ), C.POINTER(_SZ))
        self.check(f(os.fsencode(path), None, C.byref(n), C.byref(d)))
        out = np.empty((n.value, d.value))
        self.check(f(os.fsencode(path), _ptr(out), C.byref(n), C.byref(d)))
        return out

    def points_write(self, path, pts, binary=True):
        """write_points_file (io.cpp:118-126)."""
        pts = _f64(pts)
        self.check(self.fn("points_write", C.c_char_p, _P, _SZ, _SZ, _I)(os.fsencode(path), _ptr(pts), pts.shape[0],
                                                                         pts.shape[1], int(bool(binary))))

    def sample_clustered(self, n, d, c, D, r, seed):
        """sample_clustered (generators.cpp:42-106): (p, q, centers)."""
        p, q, ctr = np.empty((n, d)), np.empty((n, d)), np.empty((c, d))
        self.check(self.fn("sample_clustered", _SZ, _SZ, _SZ, C.c_double, C.c_double, _U64, _P, _P, _P)(
            n, d, c, D, r, seed, _ptr(p), _ptr(q), _ptr(ctr)))
        return p, q, ctr

    def run_all_json(self, config: dict):
        """run_all (runner.cpp:344-418) on a config_from_json dict -> records."""
        import json
        out = C.c_void_p()
        self.check(self.fn("run_all_json", C.c_char_p, C.POINTER(C.c_void_p))(json.dumps(config).encode(),
                                                                              C.byref(out)))
        try:
            return json.loads(C.string_at(out.value).decode())["records"]
        finally:
            self.fn("free_string", C.c_void_p, restype=None)(out)

    def lsh_pairs_cfg(self, p, q, scheme, bands=1, rows=1, buckets=2, iters=10, branching=2, seed=0):
        """lsh_neighbor_pairs (lsh.cpp:245-283) end to end for any scheme."""
        p, q = _f64(p), _f64(q)
        h = _P()
        self.check(self.fn("lsh_pairs_cfg", _P, _SZ, _P, _SZ, _SZ, _I, _I, _I, _I, _I, _I, _U64, _PP)(
            _ptr(p), p.shape[0], _ptr(q), q.shape[0], p.shape[1], scheme, bands, rows, buckets, iters, branching,
            seed, C.byref(h)))
        return Pairs(self, h, p.shape[0], q.shape[0])

    def sample_uniform_ball(self, n, d, seed):
        out = np.zeros((n, d))
        self.check(self.fn("sample_uniform_ball", _SZ, _SZ, _U64, _P)(n, d, seed, _ptr(out)))
        return out

    # ---- full-size parity (oracle/parity_c3.py) ---------------------------
    def hash_kmeans_band(self, all_pts, buckets, iters, seed, band):
        """One band of the k-means LSH on the union (lsh.cpp:267-281)."""
        all_pts = _f64(all_pts)
        ids = np.zeros(all_pts.shape[0], np.uint64)
        self.check(self.fn("hash_kmeans_band", _P, _SZ, _SZ, _I, _I, _U64, _I, _P)(
            _ptr(all_pts), all_pts.shape[0], all_pts.shape[1], buckets, iters, seed, band, _ptr(ids)))
        return ids

    def select_landmarks(self, p, q, l, method, seed):
        """select_landmarks (nystrom.cpp:28-48) -> l x d."""
        p, q = _f64(p), _f64(q)
        out = np.zeros((l, p.shape[1]))
        self.check(self.fn("select_landmarks", _P, _SZ, _P, _SZ, _SZ, _SZ, _I, _U64, _P)(
            _ptr(p), p.shape[0], _ptr(q), q.shape[0], p.shape[1], l, method, seed, _ptr(out)))
        return out

    def lcn_pipeline(self, p, q, kind, lam, ids_p, ids_q, range_, landmarks):
        """neighbor_pairs(BandBuckets) -> build_sparse -> build_factors ->
        build_correction -> KernelOperator::lcn; returns (Op, phase seconds)."""
        p, q, lm = _f64(p), _f64(q), _f64(landmarks)
        ids_p = np.ascontiguousarray(ids_p, np.uint64)
        ids_q = np.ascontiguousarray(ids_q, np.uint64)
        h = _P()
        ph = np.zeros(4)
        self.check(self.fn("lcn_pipeline", _P, _SZ, _P, _SZ, _SZ, _I, _D, _P, _P, _I, _U64, _P, _SZ, _P, _PP)(
            _ptr(p), p.shape[0], _ptr(q), q.shape[0], p.shape[1], kind, lam, _ptr(ids_p), _ptr(ids_q),
            ids_p.shape[0], range_, _ptr(lm), lm.shape[0], _ptr(ph), C.byref(h)))
        phases = dict(zip(["neighbor_pairs", "build_sparse", "build_factors", "build_correction"], ph / 1e3))
        return Op(self, h, p.shape[0], q.shape[0], "lcn", lm.shape[0]), phases

    def row_digest(self, op):
        """Per-row (count, sum mix64(col), xor mix64(col)) of the support."""
        cnt = np.zeros(op.n, np.uint32)
        hs = np.zeros(op.n, np.uint64)
        hx = np.zeros(op.n, np.uint64)
        self.check(self.fn("op_row_digest", _P, _P, _P, _P)(op.h, _ptr(cnt), _ptr(hs), _ptr(hx)))
        return cnt, hs, hx

    def plan_rows(self, op, res, rows, counts):
        """extract_plan entries of the listed rows: dict of cols, log_sp,
        delta, sp_vals, sp_nys_vals (flat, row after row)."""
        rows = np.ascontiguousarray(rows, np.uint32)
        tot = int(np.asarray(counts, np.int64)[rows].sum())
        cnt = np.zeros(len(rows), np.uint32)
        out = {"cols": np.zeros(tot, np.uint32)}
        for k in ("log_sp", "delta", "sp_vals", "sp_nys_vals"):
            out[k] = np.zeros(tot)
        self.check(self.fn("plan_rows", _P, _P, _P, _SZ, _P, _P, _P, _P, _P, _P)(
            op.h, res.h, _ptr(rows), len(rows), _ptr(cnt), _ptr(out["cols"]), _ptr(out["log_sp"]),
            _ptr(out["delta"]), _ptr(out["sp_vals"]), _ptr(out["sp_nys_vals"])))
        out["cnt"] = cnt
        return out


class OracleLib(CheckerLib):
    prefix = "orc_"

    def __init__(self, path=ORACLE_SO):
        super().__init__(path)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def oracle_available() -> bool:
    return os.path.exists(ORACLE_SO)
