#!/usr/bin/env python
"""Benchmark of the LCN-Sinkhorn hot path (BASELINE.json metric, configs[3]).

Metric: Sinkhorn iterations per second of LCN-Sinkhorn at n = m = 10^6,
d = 128 (configs[3]: sq-L2 / mean, lambda = 0.05, 2 x 4096 k-means LSH,
l = 512 landmarks, 100 iterations). One *step* = the 100-iteration Sinkhorn
solve on the device-resident LCN operator built from the config's seeded
synthetic points (`value`, inputs resident in HBM, timed with CUDA events on
the stream the library launches on). `e2e` is the same metric through the
C-ABI from pinned host buffers: every step copies the points and marginals
host->device, runs the *whole* reference-facing path (k-means LSH, landmarks,
Nystrom factors, LCN correction, 100 iterations) and reads the distance back;
e2e = 100 iterations / that wall of device time.

`roofline` is for the dominant kernel (band_stream_kernel), `iteration_roofline`
for one whole iteration: algorithmic bytes B_iter = 8 nnz + 4 l (n+m) +
16 (n+m) over the measured iteration time, against the
measured HBM copy bandwidth in MEASURED_PEAKS.json.

Multi-GPU (`--gpus N` spawns N ranks through torch.distributed.run; the
driver launches torchrun itself): ONE configs[3] problem, bucket-sharded
(lcn_ctx_set_comm): every rank keeps the points of its band-0 buckets (+ halo
points of later bands) and builds only their blocks and factor rows; per
half-iteration one NCCL all-gather of each rank's [low-rank partial, shift,
error, flags, halo scalings] record ("scaling": "strong"). `--replicas` runs
independent problems per GPU instead ("weak").

--impl reference times the reference's own CPU implementation (oracle/_ref:
the reference sources compiled unmodified, Nystrom restated because Eigen is
absent) on all host threads: configs[3] at scale 0.1 (bucket size, l and d
kept) built once, then each step = 5 reference Sinkhorn iterations; `value`
is the configs[3] iteration rate that implies (scaled by the iteration bytes
B_iter). The full-size reference iteration phase measured by the parity run
(profiles/parity_c3_full.json) is reported beside it.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

ITERS = 100
# what the headline arithmetic is (bench's `dtype`): delta, U and W stored in
# fp32; products and per-chunk partial sums in fp32; rows / tiles / chunks
# combined in fp64; log vectors, shifts and global reductions in fp64
DTYPE_LABEL = "f32 storage, f32 products + per-chunk partials, f64 cross-chunk accumulation and log vectors"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    FIELDS = ["index", "clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.idx)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) >= 9:
                for k, nm in enumerate(names):
                    if r[5 + k].lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref: the reference's own sources, compiled here)
# ---------------------------------------------------------------------------
REF_SAMPLE_SCALE = 0.1    # configs[3] at n = m = 1e5: 410 buckets / band (bucket size kept), l = 512; operator ~2 GB, beyond the host caches
REF_SAMPLE_ITERS = 5      # reference Sinkhorn iterations per timed step
FULL = {"n": 1_000_000, "m": 1_000_000, "d": 128, "k": 4096, "bands": 2, "l": 512, "kmeans_iters": 10}
FULL_NNZ = 521_911_712    # support of configs[3] (bucket ids bit-exact with the reference, profiles/parity_c3_full.json)


def b_iter(nnz, n, m, l):
    """SURVEY.md 8(d) bytes of one iteration: 8 nnz + 4 l (n + m) + 16 (n + m)."""
    return 8.0 * nnz + 4.0 * l * (n + m) + 16.0 * (n + m)


def workload_config():
    """The workload both arms report (same dict: the driver compares them)."""
    return {"workload": "configs[3] LCN-Sinkhorn n=m=1e6 d=128 sqL2/mean lambda=0.05 2x4096 LSH l=512",
            "n": FULL["n"], "m": FULL["m"], "d": FULL["d"], "landmarks": FULL["l"], "bands": FULL["bands"],
            "buckets": FULL["k"], "iterations_per_step": ITERS,
            "l2": "inputs larger than L2 (delta + U + W = 6.2 GB per iteration)"}


class RefSample:
    """configs[3] at REF_SAMPLE_SCALE built once by the reference's own staged
    path (k-means LSH per band -> neighbor_pairs -> select_landmarks ->
    build_factors -> build_sparse -> build_correction -> KernelOperator::lcn)
    on all host threads; each phase timed. The sample keeps configs[3]'s
    bucket size, l and d, and its operator (~1 GB) is far larger than the host
    caches, so one iteration costs what a full-size one costs per byte.
    step() times REF_SAMPLE_ITERS reference Sinkhorn iterations on it."""

    def __init__(self):
        from oracle.bindings import RefLib  # checker / baseline only
        from paper_2107_06876_b200 import configs
        self.ref = ref = RefLib()
        pr = self.pr = configs.config3(REF_SAMPLE_SCALE)
        t0 = time.perf_counter()
        ids = ref.lsh_buckets(pr.p, pr.q, pr.bands, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
        t1 = time.perf_counter()
        pairs = ref.pairs_from_buckets(ids[:, :pr.n], ids[:, pr.n:], pr.buckets)
        t2 = time.perf_counter()
        ph = [0.0] * 4
        self.op = ref.op_lcn(pr.p, pr.q, pr.cost, pr.lam_eff, pairs, pr.landmarks, 0, pr.landmark_seed, phases=ph)
        t3 = time.perf_counter()
        self.pm, self.qm = pr.marginals()
        self.nnz = int(self.op.nnz)
        self.phases = {"lsh_kmeans": t1 - t0, "lsh_pairs": t2 - t1, "landmarks": ph[0] / 1e3, "factors": ph[1] / 1e3,
                       "sparse_correction": (ph[2] + ph[3]) / 1e3, "build_wall": t3 - t0}

    def step(self, iters=REF_SAMPLE_ITERS):
        t0 = time.perf_counter()
        res = self.op.sinkhorn(self.pm, self.qm, tol=0.0, max_iters=iters, check_support=False, want_plan=False)
        dt = time.perf_counter() - t0
        assert res.iters == iters
        return dt

    def full_rate(self, sec_per_iter, full_nnz=FULL_NNZ):
        """Iterations/s at configs[3]: the sample's time per iteration scaled by
        the iteration bytes (B_iter) of the full problem."""
        pr = self.pr
        r = b_iter(full_nnz, FULL["n"], FULL["m"], FULL["l"]) / b_iter(self.nnz, pr.n, pr.m, pr.landmarks)
        return 1.0 / (sec_per_iter * r), r

    def full_solve_extrapolated(self, sec_per_iter, full_nnz=FULL_NNZ):
        """Seconds of a whole configs[3] solve (build + 100 iterations), each
        build phase scaled from the sample by its algorithmic work: k-means
        N k d per band, pairs nnz log nnz, landmarks N l, factors
        N l d + l^2 m, correction nnz l. EXTRAPOLATED (the full build is hours
        on the host; the iteration phase is measured in
        profiles/parity_c3_full.json)."""
        pr, ph = self.pr, self.phases
        N, Ns = FULL["n"] + FULL["m"], pr.n + pr.m
        l, ls = FULL["l"], pr.landmarks
        sc = {"lsh_kmeans": (N * FULL["k"]) / (Ns * pr.buckets),
              "lsh_pairs": (full_nnz * math.log2(full_nnz)) / (self.nnz * math.log2(self.nnz)),
              "landmarks": (N * l) / (Ns * ls),
              "factors": (N * l * FULL["d"] + l * l * FULL["m"]) / (Ns * ls * pr.d + ls * ls * pr.m),
              "sparse_correction": (full_nnz * l) / (self.nnz * ls)}
        parts = {k + "_s": ph[k] * sc[k] for k in sc}
        _, r = self.full_rate(sec_per_iter, full_nnz)
        parts["iterations_s"] = ITERS * sec_per_iter * r
        return sum(parts.values()), parts

    def describe(self):
        pr = self.pr
        return (f"configs[3] at scale {REF_SAMPLE_SCALE}: n=m={pr.n}, d=128, {pr.bands}x{pr.buckets} k-means LSH "
                f"(bucket size kept), l={pr.landmarks}, nnz {self.nnz}; reference build {self.phases['build_wall']:.1f}s "
                f"(untimed), then {REF_SAMPLE_ITERS} reference iterations per step; iteration time scaled to "
                f"configs[3] by the iteration bytes B_iter (x{self.full_rate(1.0)[1]:.1f})")


def full_size_measured():
    """The full-size configs[3] reference iteration phase, measured (the
    parity run, profiles/parity_c3_full.json), when present."""
    try:
        pj = json.load(open(os.path.join(ROOT, "profiles", "parity_c3_full.json")))
        r = pj.get("reference_on_gpu_box_host", pj["reference"])
        return {"iter_per_s": r["iter_per_s"], "iterations_s": r["iterations_s"], "threads": r.get("threads"),
                "host_cores": r.get("host_cores"), "where": r.get("where", "see profiles/parity_c3_full.json"),
                "build_phases_s": r.get("phases_s")}
    except Exception:
        return None


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    os.environ.setdefault("OMP_NUM_THREADS", str(cpu_cores()))
    smp = RefSample()
    for _ in range(args.warmup):
        smp.step()
    times = [smp.step() for _ in range(args.steps)]
    step_s = float(np.mean(times))
    value, ratio = smp.full_rate(step_s / REF_SAMPLE_ITERS)
    t_solve, parts = smp.full_solve_extrapolated(step_s / REF_SAMPLE_ITERS)
    cpu = {"value": value, "unit": "iter/s", "cores": cpu_cores(), "kind": "reference", "sample": smp.describe(),
           "sample_iter_per_s": REF_SAMPLE_ITERS / step_s, "sample_build_phases_s": smp.phases,
           "full_solve_s_extrapolated": t_solve, "full_solve_phases_s_extrapolated": parts,
           "full_size_measured": full_size_measured()}
    line = {"impl": "reference", "metric": "lcn_sinkhorn_iters_per_s", "value": value, "unit": "iter/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(),
            "step": f"{REF_SAMPLE_ITERS} reference iterations on the scale-{REF_SAMPLE_SCALE} sample (ms_per_step is "
                    f"that time, measured); value = the configs[3] iteration rate it implies (B_iter scaling)",
            "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def count_launches(step):
    """Kernels of ours (lcnb::) launched by one step, counted from a CUPTI
    trace of one extra, untimed step (torch.profiler)."""
    try:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step()
        names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
        return sum(1 for nm in names if "lcnb" in nm)
    except Exception:
        return None

def kernel_intervals(fn, pattern):
    """(start_us, end_us) of the CUDA kernels whose name contains `pattern`
    launched by fn(), from a CUPTI trace (torch.profiler)."""
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
    out = []
    for e in prof.events():
        if e.device_type.name == "CUDA" and pattern in e.name:
            out.append((e.time_range.start, e.time_range.end))
    return out


def union_us(iv):
    """Length of the union of intervals (kernels of concurrent jobs overlap)."""
    tot, cur_s, cur_e = 0.0, None, None
    for s_, e_ in sorted(iv):
        if cur_e is None or s_ > cur_e:
            if cur_e is not None:
                tot += cur_e - cur_s
            cur_s, cur_e = s_, e_
        else:
            cur_e = max(cur_e, e_)
    if cur_e is not None:
        tot += cur_e - cur_s
    return tot


def measure_tf32_peak(dev):
    """Dense TF32 tensor-core rate on this GPU: cuBLAS fp32 GEMM 8192^3 with
    TF32 allowed (torch.matmul), best of 10 after warm-up, CUDA events.
    MEASURED_PEAKS.json has no TF32 entry (measure it)."""
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        g = torch.Generator(device=dev).manual_seed(0)
        a = torch.randn(8192, 8192, device=dev, generator=g)
        b = torch.randn(8192, 8192, device=dev, generator=g)
        c = torch.empty(8192, 8192, device=dev)
        for _ in range(3):
            torch.matmul(a, b, out=c)
        best = float("inf")
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b, out=c)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b, c
        return 2.0 * 8192 ** 3 / (best * 1e-3) / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def distance_roofline(iv, n, m, d, bands, buckets, landmarks, iters, tf32_peak=None, point_tiles=None):
    """Tensor-core roofline of the distance blocks (the tcgen05 3xTF32
    assignment filter of the k-means in the LSH and landmark build) over the
    union of the launches' device intervals. The MMA work is what the kernel
    evaluated: the library's work counter (lcn_ctx_tc_work) of point x
    128-centroid tile products, 2 * 128 * 128 * 3 MMA flops each (hi.hi,
    hi.lo, lo.hi at 128 padded features). Lloyd's certified bounds and tile
    skipping make it data dependent; `dense_equivalent` is the work of full
    assignments of every point to every centroid."""
    N = n + m
    if d > 128 or not iv:
        return None
    # select_landmarks runs lloyd with 10 iterations (nystrom.cpp:28-48)
    launches = [buckets] * (bands * (iters + 1)) + [landmarks] * (10 + 1)
    dense_mma = sum(2.0 * N * (-(-k // 128) * 128) * 128 * 3 for k in launches)
    mma = 2.0 * 128 * 128 * 3 * point_tiles if point_tiles else None
    if mma is None:
        return None
    t = union_us(iv) * 1e-6
    nominal = 1100.0  # TF32 dense, B200_PROFILING.md
    peak = tf32_peak if tf32_peak else nominal
    kind = ("measured: cuBLAS TF32 GEMM 8192^3 (torch.matmul, allow_tf32), best of 10, this run"
            if tf32_peak else "guide (tf32 dense)")
    ach = mma / t / 1e12
    return {"bound": "tensor", "kernel": "assign_filter_tc_kernel (tcgen05.mma kind::tf32, 3xTF32)",
            "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak, "peak_kind": kind,
            "nominal_peak": nominal, "frac_vs_nominal": ach / nominal,
            "fp32_accurate_achieved": ach / 3, "fp32_accurate_peak": peak / 3,
            "launches": len(iv), "device_ms": t * 1e3, "point_tiles": point_tiles,
            "mma_flops": mma, "dense_equivalent_mma_flops": dense_mma,
            "evaluated_share_of_dense": mma / dense_mma,
            "work": "MMA flops the filter evaluated in one build (lcn_ctx_tc_work counter: point x 128-centroid "
                    "tile products x 2*128*128*3); Lloyd's bounds and tile skipping evaluate "
                    "evaluated_share_of_dense of the full assignments (bands x (iters + 1) of n+m points to the "
                    "buckets + 11 to the landmarks)"}


def batched_c4(lcn, ctx, with_cpu):
    """configs[4]: all 32768 (pair, head) problems through lcn_batched_lcn
    (host buffers in, distances out: upload, both ragged launches, the host
    factorisation and the download are inside the wall time; one untimed
    warm-up call), and the reference pipeline per problem (oracle/_ref) on a
    bounded sample of the same problems, single-threaded like the
    reference's serial loop over heads (sinkhorn.cpp:341-351)."""
    import time
    from paper_2107_06876_b200 import configs
    b = configs.config4(1.0)
    lcn.batched_lcn(ctx, b)  # warm-up
    t0 = time.perf_counter()
    dist, st, it = lcn.batched_lcn(ctx, b)
    wall = time.perf_counter() - t0
    out = {"problems": int(b.count), "problems_per_s": b.count / wall, "wall_s": wall,
           "statuses_ok": int((st == 0).sum()), "mean_distance": float(np.nanmean(dist)),
           "config": "configs[4]: 4096 pairs x 8 heads, n, m ~ U[20, 200], d = 16 after projection, L2, "
                     "lambda = 0.1, l = 10 k-means landmarks, 1 x 8 k-means LSH, 50 iterations",
           "input_bytes": int(b.X.nbytes), "launches": "2 ragged kernels (+ one per jitter retry)"}
    if with_cpu:
        try:
            from oracle.bindings import RefLib, ref_available
            if ref_available():
                import ctypes
                import threading
                ref = RefLib()
                gomp = ctypes.CDLL("libgomp.so.1")
                cores = cpu_cores()
                nxt, lock, done = [0], threading.Lock(), [0]
                t0 = time.perf_counter()

                def worker():
                    # one problem per host thread: each solve single-threaded (the
                    # reference's loop over heads is serial, sinkhorn.cpp:341-351);
                    # omp_set_num_threads sets this thread's OpenMP team size
                    gomp.omp_set_num_threads(1)
                    while True:
                        with lock:
                            k = nxt[0]
                            if k >= b.count or (time.perf_counter() - t0 > 5.0 and k >= 64 * cores):
                                return
                            nxt[0] += 1
                        p_, q_ = b.problem(k)
                        try:
                            ref.lcn_problem(p_, q_, b.cost, b.lam, b.buckets, b.kmeans_iters, b.lsh_seed(k),
                                            b.landmarks, b.landmark_seed(k), b.iters)
                        except Exception:
                            pass
                        with lock:
                            done[0] += 1

                th = [threading.Thread(target=worker) for _ in range(cores)]
                for t_ in th:
                    t_.start()
                for t_ in th:
                    t_.join()
                tw = time.perf_counter() - t0
                out["cpu_baseline"] = {"value": done[0] / tw, "unit": "problems/s", "cores": cores, "kind": "reference",
                                       "sample": f"the first {done[0]} problems of the batch on {cores} host threads "
                                                 f"(one problem per thread), {tw:.2f} s"}
        except Exception as ex:
            out["cpu_baseline"] = {"value": None, "sample": f"unavailable: {ex}"}
    return out


def dense_anchor(lcn, ctx, peak_gbs, tf32_peak=None):
    """configs[2]: the dense operator on configs[1]'s points (n = m = 20000,
    d = 300, L2, lambda = 0.05): exact fp64 log K built on the device, 50
    log-domain iterations streaming the fp32 copy (dense_lse_tma_kernel, both
    orientations), device-timed; and the approximation error of the LCN and
    sparse operators of configs[1] against its distance."""
    import torch
    from paper_2107_06876_b200 import configs
    pr = configs.config1(1.0)
    dp = torch.from_numpy(pr.p.astype(np.float32)).cuda()
    dq = torch.from_numpy(pr.q.astype(np.float32)).cuda()
    pm, qm = pr.marginals()
    op = lcn.KernelOperator.dense_device(ctx, dp.data_ptr(), pr.n, dq.data_ptr(), pr.m, pr.d, pr.cost, pr.lam_eff)
    opts = lcn.SinkhornOptions(tol=0.0, max_iters=pr.iters, want_plan=False, check_support=False)
    lcn.sinkhorn(op, pm, qm, opts)  # warm-up
    runs = [lcn.sinkhorn(op, pm, qm, opts) for _ in range(3)]
    ms_it = float(np.median([r.device_ms for r in runs])) / pr.iters
    dense_d = runs[0].distance
    b_it = 2 * 4 * pr.n * pr.m  # fp32 log K read once per half-iteration
    out = {"config": "configs[2]: dense, configs[1] points (n = m = 20000, d = 300), L2, lambda = 0.05, 50 iterations",
           "ms_per_iteration": ms_it, "iters_per_s": 1e3 / ms_it,
           "roofline": {"bound": "hbm", "achieved": b_it / (ms_it * 1e-3) / 1e9, "peak": peak_gbs, "unit": "GB/s",
                        "frac": b_it / (ms_it * 1e-3) / 1e9 / peak_gbs,
                        "algorithmic_bytes_per_iteration": b_it, "kernel": "dense_lse_tma_kernel"},
           "distance_dense": dense_d}
    del op
    # configs[2] as worded: exp(-C/lambda) recomputed every half-iteration as a
    # tcgen05 3xTF32 GEMM fused with the log-sum-exp, no n x m storage
    try:
        ctx_rc = lcn.Context(ctx.device, dense_recompute=True)
        ctx_rc.set_stream(torch.cuda.current_stream().cuda_stream)
        op_rc = lcn.KernelOperator.dense_device(ctx_rc, dp.data_ptr(), pr.n, dq.data_ptr(), pr.m, pr.d, pr.cost,
                                                pr.lam_eff)
        lcn.sinkhorn(op_rc, pm, qm, opts)
        runs_rc = [lcn.sinkhorn(op_rc, pm, qm, opts) for _ in range(3)]
        ms_rc = float(np.median([r.device_ms for r in runs_rc])) / pr.iters
        kp = -(-pr.d // 32) * 32
        mma = 2 * 2.0 * (-(-pr.n // 128) * 128) * (-(-pr.m // 128) * 128) * kp * 3  # both halves, 3 MMAs (3xTF32)
        ach = mma / (ms_rc * 1e-3) / 1e12
        out["recompute"] = {
            "what": "exp(-C/lambda) recomputed per half-iteration: tcgen05.mma kind::tf32 (3xTF32 split) dot products "
                    "+ fp64 norms, fused row / column log-sum-exp (dense_lse_tc_kernel), no n x m storage",
            "ms_per_iteration": ms_rc, "iters_per_s": 1e3 / ms_rc, "distance": runs_rc[0].distance,
            "rel_vs_stored": abs(runs_rc[0].distance - dense_d) / abs(dense_d),
            "roofline": {"bound": "tensor", "achieved": ach, "unit": "TFLOP/s", "peak": tf32_peak,
                         "frac": ach / tf32_peak if tf32_peak else None,
                         "peak_kind": "measured cuBLAS TF32 GEMM 8192^3 (this run)",
                         "mma_flops_per_iteration": mma, "kernel": "dense_lse_tc_kernel"}}
        del op_rc, runs_rc
    except Exception as ex:  # reported, never sinks the line
        out["recompute"] = {"unavailable": str(ex)}
    cfg = lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    lop = lcn.KernelOperator.lcn_lsh(ctx, pr.p, pr.q, pr.cost, pr.lam_eff, cfg, pr.landmarks, lcn.LANDMARK_KMEANS,
                                     pr.landmark_seed)
    ld = lcn.sinkhorn(lop, pm, qm, opts).distance
    out["distance_lcn"] = ld
    out["rel_error_lcn"] = abs(ld - dense_d) / abs(dense_d)
    del lop
    try:
        sop = lcn.KernelOperator.sparse_lsh(ctx, pr.p, pr.q, pr.cost, pr.lam_eff, cfg)
        sd = lcn.sinkhorn(sop, pm, qm, opts).distance
        out["distance_sparse"] = sd
        out["rel_error_sparse"] = abs(sd - dense_d) / abs(dense_d)
    except lcn.Error as ex:  # rows without LSH neighbours, as in the reference
        out["distance_sparse"] = None
        out["sparse_error"] = f"{type(ex).__name__}: {ex}"
    return out


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2107_06876_b200 as lcn
    from paper_2107_06876_b200 import configs

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    pr = configs.config3(args.scale)
    sharded = (world > 1 and not args.replicas) or args.sharded
    if rank and not sharded:
        # independent replica per rank: reseed the point draw
        import dataclasses
        rng = np.random.default_rng(2000 + rank)
        perm_p = rng.permutation(pr.n)
        pr = dataclasses.replace(pr, p=pr.p[perm_p], seed=pr.seed + rank)
    n, m, d, l = pr.n, pr.m, pr.d, pr.landmarks
    cfg = lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    stream = torch.cuda.Stream(device=dev)
    ctx = lcn.Context(local_rank)
    ctx.set_stream(stream.cuda_stream)
    if sharded:
        # one problem over all ranks (lcn_ctx_set_comm): rank 0's NCCL id
        obj = [lcn.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        ctx.set_comm(world, rank, obj[0])

    p32 = torch.from_numpy(pr.p.astype(np.float32)).pin_memory()
    q32 = torch.from_numpy(pr.q.astype(np.float32)).pin_memory()
    pm, qm = pr.marginals()
    pm_h = torch.from_numpy(pm).pin_memory()
    qm_h = torch.from_numpy(qm).pin_memory()
    opts = lcn.SinkhornOptions(tol=0.0, max_iters=ITERS, check_support=False, want_plan=False)

    with torch.cuda.stream(stream):
        dp = p32.to(dev, non_blocking=True)
        dq = q32.to(dev, non_blocking=True)
        dpm = pm_h.to(dev, non_blocking=True)
        dqm = qm_h.to(dev, non_blocking=True)
    stream.synchronize()

    # ---- build (timed once, reported as build_s) -------------------------
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    op = lcn.KernelOperator.from_device(ctx, dp.data_ptr(), n, dq.data_ptr(), m, d, pr.cost, pr.lam_eff, cfg, l,
                                        lcn.LANDMARK_KMEANS, pr.landmark_seed)
    e1.record(stream)
    stream.synchronize()
    build_ms = e0.elapsed_time(e1)
    nnz = op.nnz
    stored = op.stored
    streamed = op.streamed

    def step():
        r = lcn.sinkhorn_device(op, dpm.data_ptr(), dqm.data_ptr(), opts)
        return r

    for _ in range(args.warmup):
        res = step()
    launches_per_step = count_launches(step)

    clocks = Clocks(int(os.environ.get("LCN_GPU_INDEX", local_rank)))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        res = step()
    t1.record(stream)
    torch.cuda.synchronize()
    # kernel durations: a second timed region of the same K steps with phase
    # events recorded by the library on its own stream between its launches
    # (kept out of the region `value` is measured on: ~4% event overhead)
    ctx.set_profile(True)
    phase_ms, phase_it = [0.0] * 4, 0
    for _ in range(args.steps):
        r_ = step()
        pm_, it_ = r_.phase_ms()
        phase_ms = [a_ + b_ for a_, b_ in zip(phase_ms, pm_)]
        phase_it += it_
        del r_
    ctx.set_profile(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    elapsed = t0.elapsed_time(t1) / 1e3  # s
    if world > 1:
        tt = torch.tensor([elapsed], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed = float(tt.item())
    ms_per_step = elapsed * 1e3 / args.steps
    # replicas: every rank solves its own problem; sharded: the ranks solve one
    value = (1 if sharded else world) * ITERS * args.steps / elapsed
    distance = res.distance / pr.mu

    # ---- roofline ------------------------------------------------------------
    # Dominant kernel: band_stream_kernel (2 bands x {row, column} pass launches
    # per iteration). Algorithmic bytes per iteration:
    #   delta over the support, fp32, read once per pass: 8 nnz
    #   per band and pass one fp64 scaling vector in + one fp64 correction out:
    #   16 (n + m) per band
    # divided by the band launches' time, from the live phase events.
    hbm, peak_kind = peaks()
    per_it = {k: v / max(phase_it, 1) for k, v in
              zip(["col_bands", "col_finalize", "row_bands", "row_finalize"], phase_ms)}
    band_launches = 2 * pr.bands
    a_band = 8 * nnz + 16 * pr.bands * (n + m)
    if sharded:  # this rank streams about 1/world of the band blocks
        a_band /= world
    t_band = (per_it["row_bands"] + per_it["col_bands"]) / 1e3  # s per iteration
    achieved = (a_band / band_launches) / (t_band / band_launches) / 1e9
    traffic = None
    prof_path = os.path.join(ROOT, "profiles", "band_traffic.json")
    if os.path.exists(prof_path):
        try:
            tj = json.load(open(prof_path))
            if tj.get("nnz") == nnz:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    # whole iteration (SURVEY.md 8(d) B_iter)
    b_iter = 8 * nnz + 4 * l * (n + m) + 16 * (n + m)
    t_iter = (ms_per_step / 1e3) / ITERS
    it_achieved = b_iter / t_iter / 1e9

    # ---- fp64 storage (LCN_STORE_FP64: the reference's precision) -------------
    fp64_line = None
    if not args.no_fp64:
        del op
        torch.cuda.synchronize()
        ctx64 = lcn.Context(local_rank, store_fp64=True)
        ctx64.set_stream(stream.cuda_stream)
        if sharded:  # a fresh NCCL id per communicator
            obj64 = [lcn.nccl_unique_id() if rank == 0 else None]
            if world > 1:
                dist.broadcast_object_list(obj64, src=0)
            ctx64.set_comm(world, rank, obj64[0])
        op64 = lcn.KernelOperator.from_device(ctx64, dp.data_ptr(), n, dq.data_ptr(), m, d, pr.cost, pr.lam_eff, cfg, l,
                                              lcn.LANDMARK_KMEANS, pr.landmark_seed)
        k64 = max(3, min(args.steps, 5))
        r64 = lcn.sinkhorn_device(op64, dpm.data_ptr(), dqm.data_ptr(), opts)  # warm-up
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a64, b64 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a64.record(stream)
        for _ in range(k64):
            r64 = lcn.sinkhorn_device(op64, dpm.data_ptr(), dqm.data_ptr(), opts)
        b64.record(stream)
        torch.cuda.synchronize()
        el64 = a64.elapsed_time(b64) / 1e3
        if world > 1:
            tt = torch.tensor([el64], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            el64 = float(tt.item())
        t_it64 = el64 / (k64 * ITERS)
        b_iter64 = 16 * nnz + 8 * l * (n + m) + 16 * (n + m)
        fp64_line = {"value": (1 if sharded else world) * ITERS * k64 / el64, "unit": "iter/s", "steps": k64,
                     "ms_per_iteration": t_it64 * 1e3, "distance": r64.distance / pr.mu,
                     "dtype": "f64 storage and arithmetic (LCN_STORE_FP64)",
                     "iteration_roofline": {"bound": "hbm", "achieved": b_iter64 / t_it64 / 1e9, "peak": hbm,
                                            "unit": "GB/s", "frac": b_iter64 / t_it64 / 1e9 / hbm,
                                            "algorithmic_bytes_per_iteration": b_iter64}}
        del r64, op64
        ctx64.close()
        torch.cuda.synchronize()

    # ---- e2e through the reference-facing C-ABI from pinned host buffers -------
    # lcn_op_lcn_lsh (fp64 host points, as the reference's PointSet) + lcn_sinkhorn
    # (host marginals, Marginals::validate on the host, no plan): the call a
    # caller of lsh_neighbor_pairs / select_landmarks / build_factors /
    # build_correction / sinkhorn makes
    e2e = None
    dist_roof = None
    dist_iv = None
    dist_tiles = None
    if not args.no_e2e:
        if fp64_line is None:
            del op
        torch.cuda.synchronize()
        p64 = torch.from_numpy(pr.p).pin_memory().numpy()
        q64 = torch.from_numpy(pr.q).pin_memory().numpy()
        pm64 = torch.from_numpy(pm).pin_memory().numpy()
        qm64 = torch.from_numpy(qm).pin_memory().numpy()
        h2d = int(p64.nbytes + q64.nbytes + pm64.nbytes + qm64.nbytes)
        tot = 0.0
        # untimed warm-up solves (first-use costs: pool growth), then e2e_steps timed ones
        for it in range(args.e2e_warmup + args.e2e_steps):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)

            def build2():
                return lcn.KernelOperator.lcn_lsh(ctx, p64, q64, pr.cost, pr.lam_eff, cfg, l, lcn.LANDMARK_KMEANS,
                                                  pr.landmark_seed)
            if it == 0 and args.e2e_warmup > 0:
                # the untimed warm-up build doubles as the tensor-core trace
                holder = []
                try:
                    ctx.tc_work(reset=True)
                    iv = kernel_intervals(lambda: holder.append(build2()), "assign_filter_tc_kernel")
                    dist_iv = iv  # roofline computed after the timed regions (TF32 peak GEMM)
                    dist_tiles = ctx.tc_work(reset=True)
                except Exception as ex:  # profiler unavailable: report none
                    print("distance roofline unavailable:", ex, file=sys.stderr)
                op2 = holder[0] if holder else build2()
            else:
                op2 = build2()
            r2 = lcn.sinkhorn(op2, pm64, qm64, opts)  # distance read back to the host (8 B)
            _ = r2.distance
            b.record(stream)
            torch.cuda.synchronize()
            dt = a.elapsed_time(b) / 1e3
            if world > 1:
                tt = torch.tensor([dt], device=dev, dtype=torch.float64)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                dt = float(tt.item())
            if it >= args.e2e_warmup:
                tot += dt
            del op2, r2
        e2e = {"value": (1 if sharded else world) * ITERS * args.e2e_steps / tot, "unit": "iter/s",
               "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": 8, "solve_s": tot / args.e2e_steps, "steps": args.e2e_steps,
               "warmup": args.e2e_warmup, "entry": "lcn_op_lcn_lsh + lcn_sinkhorn (host fp64 buffers, pinned)",
               "covers": "H2D fp64 points + marginals, k-means LSH, landmarks, Nystrom, correction, 100 iterations, "
                         "D2H distance"}

    # ---- CPU baseline (rank 0, N = 1) ------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            os.environ.setdefault("OMP_NUM_THREADS", str(cpu_cores()))
            smp = RefSample()
            smp.step()  # warm-up
            st_ = float(np.mean([smp.step() for _ in range(3)]))
            v_, _ = smp.full_rate(st_ / REF_SAMPLE_ITERS, nnz if args.scale == 1.0 else FULL_NNZ)
            cpu = {"value": v_, "unit": "iter/s", "cores": cpu_cores(), "kind": "reference", "sample": smp.describe(),
                   "sample_iter_per_s": REF_SAMPLE_ITERS / st_, "full_size_measured": full_size_measured()}
            del smp
        except Exception as ex:  # the baseline must never sink the GPU line
            cpu = {"value": None, "unit": "iter/s", "cores": cpu_cores(), "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    c4 = None
    if rank == 0 and world == 1 and not args.no_c4:
        try:
            c4 = batched_c4(lcn, ctx, not args.no_cpu)
        except Exception as ex:
            c4 = {"unavailable": str(ex)}
    tf32 = None
    if dist_iv is not None or not args.no_dense:
        try:
            tf32 = measure_tf32_peak(dev)
        except Exception as ex:
            print("tf32 peak measurement failed:", ex, file=sys.stderr)
        if dist_iv is not None:
            dist_roof = distance_roofline(dist_iv, n, m, d, pr.bands, pr.buckets, l, pr.kmeans_iters, tf32, dist_tiles)
    anchor = None
    if rank == 0 and not args.no_dense:
        try:
            anchor = dense_anchor(lcn, ctx, hbm, tf32)
        except Exception as ex:
            anchor = {"unavailable": str(ex)}
    sparse_op = None
    if rank == 0 and world == 1 and not args.no_dense:
        # KernelOperator::sparse (configs[0]'s operator) on configs[3]'s LSH support:
        # the log-domain band passes, fp32 log K both orientations
        try:
            sop = lcn.KernelOperator.from_device(ctx, dp.data_ptr(), n, dq.data_ptr(), m, d, pr.cost, pr.lam_eff, cfg, 0)
            sopts = lcn.SinkhornOptions(tol=0.0, max_iters=ITERS, check_support=False, want_plan=False)
            lcn.sinkhorn_device(sop, dpm.data_ptr(), dqm.data_ptr(), sopts)
            rs = [lcn.sinkhorn_device(sop, dpm.data_ptr(), dqm.data_ptr(), sopts) for _ in range(3)]
            ms_s = float(np.median([r_.device_ms for r_ in rs])) / ITERS
            b_s = 8.0 * sop.nnz + 32.0 * (n + m)
            sparse_op = {"config": "KernelOperator::sparse on configs[3]'s 2 x 4096 k-means LSH support, 100 iterations",
                         "ms_per_iteration": ms_s, "iters_per_s": 1e3 / ms_s, "nnz": sop.nnz,
                         "roofline": {"bound": "hbm", "achieved": b_s / (ms_s * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                                      "frac": b_s / (ms_s * 1e-3) / 1e9 / hbm,
                                      "algorithmic_bytes_per_iteration": b_s,
                                      "kernel": "band_stream_kernel, log-sum-exp mode (row and column band passes, single-read online consumer)"}}
            del sop, rs
        except Exception as ex:
            sparse_op = {"unavailable": str(ex)}

    gpu_launches = args.steps * launches_per_step if launches_per_step else None
    if rank == 0:
        line = {"metric": "lcn_sinkhorn_iters_per_s", "value": value, "unit": "iter/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong" if sharded else "weak", "vs_baseline": None,
                "dtype": DTYPE_LABEL, "data": "synthetic",
                "config": (workload_config() if args.scale == 1.0 else
                           dict(workload_config(), workload=f"configs[3] at scale {args.scale}", n=n, m=m,
                                landmarks=l, buckets=pr.buckets)),
                "layout": {"nnz": nnz, "stored_entries": stored, "streamed_entries": streamed,
                           "stored_entries_this_rank": stored},
                "parallelism": (f"one problem bucket-sharded over {world} GPUs: each rank owns the points of its "
                                f"band-0 buckets (+ halo of later bands) and builds only their blocks and factor rows; "
                                f"per half-iteration one NCCL all-gather of the [low-rank partial, shift, error, "
                                f"flags, halo scalings] records" if sharded else
                                f"{world} independent replica(s), 1 per GPU"),
                "distance": distance, "build_s": build_ms / 1e3,
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                             "frac": achieved / hbm, "traffic": traffic, "peak_kind": peak_kind,
                             "kernel": "band_stream_kernel (row + column band passes)",
                             "algorithmic_bytes_per_launch": a_band / band_launches,
                             "launches_per_iteration": band_launches,
                             "avg_launch_ms": t_band * 1e3 / band_launches,
                             "share_of_iteration": t_band / t_iter},
                "iteration_roofline": {"bound": "hbm", "achieved": it_achieved, "peak": hbm, "unit": "GB/s",
                                       "frac": it_achieved / hbm, "algorithmic_bytes_per_iteration": b_iter,
                                       "ms_per_iteration": t_iter * 1e3},
                "distance_roofline": dist_roof,
                "batched_c4": c4,
                "dense_anchor": anchor,
                "sparse_operator": sparse_op,
                "phases_ms_per_iteration": per_it,
                "fp64_storage": fp64_line,
                "clocks": clk, "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": gpu_launches}
        emit(line)
    return 0


_OUT_FD = None


def spawn_ranks(n):
    """`python bench.py --gpus N` outside torchrun: re-launch this command as
    N ranks (one process per GPU) through torch.distributed.run on 127.0.0.1,
    the way the driver launches it, with NCCL's init lines on stderr."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    print("bench: spawning", " ".join(cmd), file=sys.stderr, flush=True)
    # rank 0 writes the JSON line to its stdout; pass the original stdout through
    return subprocess.call(cmd, env=env, stdout=_OUT_FD if _OUT_FD is not None else None)


def emit(line):
    """Write the one JSON line to the original stdout (everything else, e.g.
    NCCL's version banner, goes to stderr)."""
    data = (json.dumps(line) + "\n").encode()
    os.write(_OUT_FD if _OUT_FD is not None else 1, data)


def main():
    global _OUT_FD
    # libraries (NCCL banners, ...) print to fd 1: send fd 1 to stderr and keep
    # the original stdout for the JSON line
    sys.stdout.flush()
    _OUT_FD = os.dup(1)
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--e2e-warmup", type=int, default=2)
    ap.add_argument("--no-c4", action="store_true", help="skip the configs[4] batched-problems line")
    ap.add_argument("--no-dense", action="store_true", help="skip the configs[2] dense-anchor object")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fp64", action="store_true", help="skip the LCN_STORE_FP64 iteration line")
    ap.add_argument("--dry-run", action="store_true", help="print the rank layout and exit (launch check)")
    ap.add_argument("--sharded", action="store_true",
                    help="use the sharded solve even on one GPU (1-rank communicator)")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent problems per GPU instead of one sharded problem")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dry_run:  # launch check only: which rank am I, out of how many
        if rank == 0 or world == 1:
            emit({"dry_run": True, "n_gpus": world, "rank": rank, "local_rank": local_rank})
        return 0
    if args.impl == "reference":
        return run_reference(args, rank, world)
    # our device pool: map 64 GB up front (the library's allocations are then
    # carved from resident memory; see lcn_ctx_create) -- the configs[3]
    # build + solve peaks well below that on a 180 GB B200
    os.environ.setdefault("LCN_POOL_RESERVE_GB", "64")
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # NCCL's init lines (rings, NVLS) go to stderr
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        return run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
