#!/usr/bin/env python
"""Benchmark: one step = one complete adaptive H^2 construction (Algorithm 1, all SURVEY §8(a)
rows: Omega, dense-kernel sketch, D/B generation, BSR subtraction, CPQR convergence test / ID,
shrink / upsweep, adaptive sample growth) of the BASELINE workload.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload NAME]

Default workload = BASELINE.json configs[1]: 3D exp covariance (l = 0.2), N = 2^18 uniform points,
leaf 64, eta 0.7, tol 1e-6, dense-kernel sketch, adaptive d_init = d_blk = 32.  Metric = build
time in seconds (lower is better) + samples used.  N > 1 GPUs (torchrun): the sketch rows are
sharded over ranks (h2_dense_sketch on the rank's rows) and all-gathered with NCCL inside the
sketch callback; the O(N) construction proper runs replicated.
--impl reference times the CPU oracle (oracle/) on a bounded sample of the same workload.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "H2 build time (s) + samples used vs N at tol=1e-6"
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 64 FP64 FMA/clk/SM (DFMA = DMMA pipe), 1965 MHz
FP64_PIPE_TOPS = 148 * 64 * 1.965e9 / 1e12          # FP64 pipe instructions (lane-ops) per second
F_EVAL = 18   # FP64 pipe ops per kernel entry in sketch_tc_kernel (SASS: 6 r^2, 5 r, 6 exp (1024-entry table,
              # degree-3 polynomial), 1 fixed-point DFMA); 19 with the round-1 256-entry / degree-4 form
F_EVAL_HELM = 27   # Helmholtz entry (SASS): 6 r^2, 5 1/r', 1 r', 4 reduction, 1 g^2, 2 c, 3 s, 2 C c - S s, 2 v, 1 w
INT8_DENSE_TOPS = 4500.0                            # nominal dense int8 tensor ops/s (B200, guide)
# measured int8 tcgen05 rate at the sketch's shape (M = 128, N = 160, K = 32, smem operands):
# profiles/r2_mma_overlap.txt (tools/microbench/mma_fp64_overlap.cu)
INT8_MEASURED_TOPS = 4307.5
FP64_DFMA_TFLOPS = 37.0   # measured DFMA (profiles/r2_fp64_mix.txt: 64 lane-ops/clk/SM; r1: 37.0 TF/s)


def hbm_peak():
    """HBM copy bandwidth (GB/s): the driver-written MEASURED_PEAKS.json, else the profiling guide's
    fallback (6.65 TB/s)."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "MEASURED_PEAKS.json"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def torch_kx_rows(Xt, kind, param, P, rows, blk=256):
    """Independent verification reference (untimed): K(rows, :) @ P with plain torch FP64 ops on
    the GPU -- elementwise r = ((dx^2 + dy^2) + dz^2)^(1/2), exp(-r/l) or cos(k r)/r (0 at r = 0),
    then a DGEMM.  Neither libh2 nor oracle/ (bench.py touches oracle/ only in its cpu_baseline /
    reference legs).  Xt: n x dim tree-ordered points (host), P: n x q (device), rows: sorted
    int array (host)."""
    import torch
    X = torch.from_numpy(np.ascontiguousarray(Xt)).cuda()
    out = []
    for a in range(0, len(rows), blk):
        Q = X[torch.from_numpy(rows[a:a + blk]).cuda()]
        r2 = (Q[:, None, 0] - X[None, :, 0]) ** 2
        for ax in range(1, X.shape[1]):
            r2 += (Q[:, None, ax] - X[None, :, ax]) ** 2
        r = torch.sqrt_(r2)
        if kind == "exp":
            K = torch.exp(-r / param)
        else:
            K = torch.where(r > 0, torch.cos(param * r) / torch.where(r > 0, r, 1.0), 0.0)
        out.append(K @ P)
        del r2, r, K
    return torch.cat(out).cpu().numpy()


def whole_build_roofline(stats, ms, n, rows_local, sk_launches, ncol_launch, slices, f_eval=F_EVAL):
    """T* = sum over phases of max(F / P_fp64, B / P_hbm) over the ALGORITHMIC work
    libh2 counts (h2_build_stats.work_flops / work_bytes), plus the dense sketch at its serialised
    bound (FP64 evaluation + int8 contraction: the two do not overlap on an SM,
    profiles/r2_sketch_serialization.md); frac = T* / measured build time."""
    hbm, hbm_src = hbm_peak()
    p64 = FP64_DFMA_TFLOPS * 1e12
    phases = {}
    for ph in ("rand", "gen", "bsr", "cpqr", "id"):
        F, B = stats["work_flops"][ph], stats["work_bytes"][ph]
        t = max(F / p64, B / (hbm * 1e9)) * 1e3
        phases[ph] = {"flops": F, "bytes": B, "t_star_ms": round(t, 3),
                      "bound": "fp64" if F / p64 >= B / (hbm * 1e9) else "hbm",
                      "measured_ms": round(stats["t_phase_ms"][ph], 3)}
    ent = float(rows_local) * n * sk_launches
    t_fp64 = ent * f_eval / (FP64_PIPE_TOPS * 1e12) * 1e3
    t_i8 = ent * ncol_launch * slices * 2 / (INT8_MEASURED_TOPS * 1e12) * 1e3
    phases["sketch"] = {"fp64_ops": ent * f_eval, "int8_ops": ent * ncol_launch * slices * 2,
                        "t_fp64_ms": round(t_fp64, 2), "t_int8_ms": round(t_i8, 2), "t_star_ms": round(t_fp64 + t_i8, 2),
                        "bound": "fp64 + int8 (serialised)", "measured_ms": round(stats["t_phase_ms"]["sketch"], 3)}
    tstar = sum(v["t_star_ms"] for v in phases.values())
    return {"t_star_ms": round(tstar, 2), "measured_ms": round(ms, 2), "frac": tstar / ms,
            "peaks": {"fp64_tflops": FP64_DFMA_TFLOPS, "hbm_gbs": hbm, "hbm_source": hbm_src,
                      "int8_tops": INT8_MEASURED_TOPS, "fp64_pipe_tops": FP64_PIPE_TOPS},
            "phases": phases,
            "note": "construction phases: libh2's algorithmic work counters (BSR 2 nc sum rows x cols, CPQR "
                    "sum 4(d-i)(m-i), ID k^2(m-k) + shrink 2k(m-k)nc, gen 8 B per stored entry); sketch: N^2 x "
                    f"{f_eval} FP64 ops + the exact int8 contraction at the measured tcgen05 rate, serialised"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default="cov3d_256k")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    p.add_argument("--no-c3", action="store_true", help="skip the N = 2^21 (configs[2]) extra timing")
    return p.parse_args()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def workload_cfg(name):
    from synth import WORKLOADS
    w = dict(WORKLOADS[name])
    return w


# ------------------------------------------------------------------------------------------
# reference arm / cpu_baseline: the C oracle (oracle/c/h2oracle.c, OpenMP on the host cores)
# ------------------------------------------------------------------------------------------
SKETCH_SAMPLE_ROWS = 128   # rows of the oracle's own dense sketch timed per step (scaled by N / rows)
TABLE_COLS = 256           # sketch columns supplied as a table to the oracle's construction proper


class OracleSetup:
    """Untimed set-up of the oracle timing (SURVEY §8(d) "Oracle timing"): the oracle's own
    KD-tree and partition (oracle/geometry.py), and the sketch Y = K Omega of the first
    TABLE_COLS columns of the Omega stream as a TABLE (data shared, code not: computed by plain
    torch FP64 -- elementwise distances, exp, DGEMM -- on the GPU when present; no libh2 code),
    so that the oracle's construction proper runs on the real sketch of the workload
    with its own adaptive loop and sample count."""

    def __init__(self, w, X, table=True):
        from oracle import geometry, c_h2
        self.c_h2 = c_h2
        t0 = time.perf_counter()
        self.tree = geometry.build_cluster_tree(X, w["leaf"])
        self.part = geometry.build_partition(self.tree, 0.7)
        self.ta = c_h2.TreeArrays(self.tree, self.part, X)
        self.w = w
        self.n = X.shape[0]
        self.Om = c_h2.omega(1, 0, 0, self.n, 0, TABLE_COLS)
        self.Y = self._table() if table else None
        self.setup_s = time.perf_counter() - t0

    def _table(self):
        import torch
        dev = "cuda" if torch.cuda.is_available() else "cpu"
        P = torch.from_numpy(self.ta.pts).to(dev)
        Om = torch.from_numpy(self.Om).to(dev)
        Y = torch.empty((self.n, TABLE_COLS), dtype=torch.float64, device=dev)
        blk = 4096 if dev == "cuda" else 256
        kind, p = self.w["kernel"], self.w["param"]
        for r0 in range(0, self.n, blk):
            Q = P[r0:r0 + blk]
            # r^2 = (dx*dx + dy*dy) + dz*dz elementwise (no |x|^2 + |y|^2 - 2xy cancellation)
            r2 = (Q[:, None, 0] - P[None, :, 0]) ** 2
            r2 += (Q[:, None, 1] - P[None, :, 1]) ** 2
            r2 += (Q[:, None, 2] - P[None, :, 2]) ** 2
            r = torch.sqrt_(r2)
            if kind == "exp":
                K = torch.exp(-r / p)
            else:
                K = torch.where(r > 0, torch.cos(p * r) / torch.where(r > 0, r, 1.0), 0.0)
            Y[r0:r0 + blk] = K @ Om
            del r, K
        out = Y.cpu().numpy()
        del Y, Om, P
        if dev == "cuda":
            torch.cuda.empty_cache()
        return out

    def step(self, threads=0):
        """One reference step: (a) the oracle's construction proper (Algorithm 1 after the sketch:
        D/B generation, BSR, CPQR convergence tests, updateSamples replays, ID, shrink, projection,
        every level) on the table, measured in full; (b) the oracle's own dense sketch for the
        draws its adaptive loop made (d_init, then d_blk per extra round), timed on
        SKETCH_SAMPLE_ROWS rows and scaled by N / rows (every row costs the same N kernel
        evaluations and N x nc multiply-adds).  Returns seconds (construction + extrapolated
        sketch) and the details."""
        c_h2, w = self.c_h2, self.w
        opts = dict(d_init=32, d_blk=32, d_max=512, threads=threads)
        R = c_h2.build(self.ta, w["kernel"], w["param"], w["tol"], y_table=self.Y, **opts)
        t_cons = R.seconds["total"] - R.seconds["sketch"]          # table copies are not sketch work
        draws = [(0, 32)] + [(c0, 32) for c0 in range(32, R.samples, 32)]
        r0 = self.n // 2 - SKETCH_SAMPLE_ROWS // 2
        t_sk = 0.0
        for c0, nc in draws:
            Om = np.ascontiguousarray(self.Om[:, c0:c0 + nc])
            t1 = time.perf_counter()
            c_h2.dense_sketch(self.ta, w["kernel"], w["param"], Om, rows=(r0, r0 + SKETCH_SAMPLE_ROWS))
            t_sk += time.perf_counter() - t1
        factor = self.n / SKETCH_SAMPLE_ROWS
        return t_cons + t_sk * factor, {"construction_s": t_cons, "sketch_sample_s": t_sk, "sketch_factor": factor,
                                        "sketch_extrapolated_s": t_sk * factor, "samples": R.samples,
                                        "draws": len(draws), "phase_s": {k: round(v, 4) for k, v in R.seconds.items()}}


def oracle_c1_seconds():
    """BASELINE configs[0] (C1): the full C oracle (own sketch) end to end, all threads and one
    thread; median of 3."""
    from oracle import geometry, c_h2
    from synth import WORKLOADS
    w = WORKLOADS["cov2d_1k"]
    X = w["points"]()
    tree = geometry.build_cluster_tree(X, w["leaf"])
    ta = c_h2.TreeArrays(tree, geometry.build_partition(tree, 0.7), X)
    out = {}
    for th, name in ((0, "all_threads_s"), (1, "one_thread_s")):
        c_h2.build(ta, "exp", 0.2, 1e-6, threads=th)
        out[name] = float(statistics.median(c_h2.build(ta, "exp", 0.2, 1e-6, threads=th).seconds["total"]
                                            for _ in range(3)))
    out["samples"] = c_h2.build(ta, "exp", 0.2, 1e-6).samples
    return out


def cpu_baseline_record(value, info, setup, steps_timed, cores):
    return {"value": value, "unit": "s", "cores": cores, "kind": "extrapolated",
            "sample": (f"per step: the C oracle's construction proper on the FULL workload (all levels, its own "
                       f"adaptive loop: {info['samples']} samples) on the sketch supplied as a table, measured "
                       f"({info['construction_s']:.2f} s), + its own dense sketch for its {info['draws']} draws timed "
                       f"on {SKETCH_SAMPLE_ROWS} rows ({info['sketch_sample_s']:.2f} s) x N/rows = "
                       f"{info['sketch_factor']:.0f} (extrapolated {info['sketch_extrapolated_s']:.1f} s)"),
            "timed_s_per_step": info["construction_s"] + info["sketch_sample_s"],
            "construction_s": info["construction_s"], "sketch_extrapolated_s": info["sketch_extrapolated_s"],
            "extrapolation_factor_sketch": info["sketch_factor"], "oracle_samples": info["samples"],
            "oracle_phase_s": info["phase_s"], "setup_untimed_s": round(setup.setup_s, 1),
            "steps_timed": steps_timed}


def run_reference(args, w, rank):
    if rank != 0:
        return
    from oracle import c_h2
    X = w["points"]()
    cores = c_h2.max_threads()
    setup = OracleSetup(w, X)
    for _ in range(min(args.warmup, 1)):   # warm-up: one untimed step (page-in, thread pool)
        setup.step()
    vals, info = [], None
    for _ in range(args.steps):
        v, info = setup.step()
        vals.append(v)
    value = float(statistics.median(vals))
    cpu = cpu_baseline_record(value, info, setup, args.steps, cores)
    cpu["c1_full_oracle"] = oracle_c1_seconds()
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": args.workload, "n": int(X.shape[0]), "leaf": w["leaf"], "eta": 0.7, "tol": w["tol"],
                      "kernel": f"{w['kernel']}({w['param']})", "sketch": "dense-kernel", "d_init": 32, "d_blk": 32,
                      "d_max": 512},
           "cpu_baseline": cpu,
           "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------
def run_ours(args, w, rank, world, local_rank):
    import torch
    import paper_2506_16759_b200 as g
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    X = w["points"]()
    n = X.shape[0]
    kern = (w["kernel"], w["param"])
    T = g.Tree(X, w["leaf"], 0.7)
    opts = dict(adaptive=True, d_init=32, d_blk=32, d_max=512)
    dist = None
    comm = None
    if world > 1:
        # sharded construction (h2_build_dist, S§8(e)): every rank owns a subtree range per
        # level, sketch rows of its leaves, its blocks; per-level NCCL all-gathers of ranks,
        # skeleton indices and Omega rows
        import torch.distributed as dist
        from paper_2506_16759_b200.dist import Comm, NcclComm
        # NCCL: libh2's in-library communicator (h2_comm_init, stream-ordered broadcast groups);
        # gloo (ranks sharing one GPU): the torch.distributed callback communicator
        comm = NcclComm() if dist.get_backend() == "nccl" else Comm()

    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)   # > L2 (126 MB)
    stream = torch.cuda.current_stream()

    def one():
        return g.build(T, kern, w["tol"], comm=comm, **opts)

    for _ in range(args.warmup):
        H = one()
        del H
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    times, stats = [], []
    for _ in range(args.steps):
        flush.fill_(1.0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        H = one()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        stats.append(H.stats)
        if _ != args.steps - 1:
            del H
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    ms = float(np.mean(times))
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    st = stats[-1]
    if comm is not None:
        H.allgather(comm)   # untimed: complete every rank's copy for the verification matvec
    # verification (untimed): dense probes  ||H X - K X||_F / ||K X||_F
    Xp = torch.from_numpy(np.random.default_rng(2).standard_normal((n, 16))).to(dev)
    KX = g.dense_sketch(T, Xp, kern)
    HX = H.matvec(Xp)
    verr = float(torch.linalg.norm(HX - KX) / torch.linalg.norm(KX))
    vrows = np.sort(np.random.default_rng(9).choice(n, 256, replace=False))
    KXt = torch_kx_rows(X[T.perm], w["kernel"], w["param"], Xp, vrows)
    verr_t = float(np.linalg.norm(HX.cpu().numpy()[vrows] - KXt) / np.linalg.norm(KXt))
    # the paper's own measure: ||H - K||_2 / ||K||_2 by power iterations
    # (h2_verify_2norm; one-column FP64 DMMA sketches, ~0.1 s each at N = 2^18; untimed)
    p2 = H.verify_2norm(kern, iters=8, nvec=8) if n <= (1 << 18) else None
    # roofline of the dominant kernel (sketch_tc_kernel, one launch per 160-column pass): the
    # contraction runs exactly on the int8 tensor cores, so the bound is the FP64 pipe evaluating
    # K: algorithmic work = N_rows * N entries x F_EVAL FP64 ops per launch
    sk_launches = st["entries_sketch"] // (n * n)
    ncol_launch = -(-st["sketch_columns"] // max(sk_launches, 1))
    slices = 7 if os.environ.get("H2_TC_SLICES") == "7" else 6   # libh2's fixed-point byte slices
    ncol_launch = min(160 if slices == 6 else 128, -(-ncol_launch // 32) * 32)
    t_sk_ms = float(np.mean([s["t_phase_ms"]["sketch"] for s in stats]))
    per_launch_ms = t_sk_ms / max(sk_launches, 1)
    rows_local = n if world == 1 else (n // world)
    entries_launch = float(rows_local) * n
    achieved = entries_launch * F_EVAL / (per_launch_ms * 1e-3) / 1e12
    int8_ops = entries_launch * ncol_launch * slices * 2 / (per_launch_ms * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r2_sketch_tc_traffic.json")
    if os.path.exists(tpath) and args.workload == "cov3d_256k" and world == 1:
        traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
    # e2e through the public API from host buffers: tree build + H2D + build + D2H of skeletons
    e2e = None
    if not args.no_e2e:
        Xpin = torch.from_numpy(X).pin_memory()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e_times, d2h = [], 0
        for it in range(1 + max(1, min(args.steps, 3))):   # iteration 0: untimed warm-up
            t0 = time.perf_counter()
            # asynchronous partition: the host's dual traversal overlaps the first sketch pass
            T2 = g.Tree(Xpin.numpy(), w["leaf"], 0.7, asynchronous=True)
            H2 = g.build(T2, kern, w["tol"], comm=comm, **opts)
            rk, sk = H2.ranks_and_skeletons()   # the result read: ranks + skeletons, every depth
            d2h = rk.nbytes + sk.nbytes
            torch.cuda.synchronize()
            if it:
                e_times.append(time.perf_counter() - t0)
            del H2, T2
        e_s = float(np.mean(e_times))
        if dist:
            t = torch.tensor([e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_s = float(t.item())
        e2e = {"value": e_s, "unit": "s", "h2d_bytes_per_step": int(X.nbytes), "d2h_bytes_per_step": int(d2h),
               "note": "wall clock incl. the coordinate upload, the KD ordering (on the GPU: radix sorts per depth, "
                       "h2_tree_build_async), the block partition (host thread, overlapped with the first sketch "
                       "pass), h2_build, D2H of ranks+skeletons"}
    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu:
        from oracle import c_h2
        setup = OracleSetup(w, X)
        v, info = setup.step()
        cpu = cpu_baseline_record(v, info, setup, 1, c_h2.max_threads())
    out = {
        "metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "n": n, "leaf": w["leaf"], "eta": 0.7, "tol": w["tol"],
                   "kernel": f"{w['kernel']}({w['param']})", "sketch": "dense-kernel (row shards)" if world > 1
                   else "dense-kernel", "d_init": 32, "d_blk": 32, "d_max": 512,
                   "eps_rule": "s*tol*rho*gamma^(Dl-t), s=0.04, gamma=1.25 (DESIGN.md R31)",
                   "sketch_format": "int8 tcgen05, 6-byte fixed-point K (2^-47 grid), 160-column pass (R32)",
                   "parallelism": (f"subtree shards x{world} (sketch rows, clusters per level; "
                                   f"{'in-library NCCL' if dist and dist.get_backend() == 'nccl' else 'gloo'} "
                                   f"all-gathers of ranks / skeletons + halo all-to-all of Omega rows"
                                   f"{'' if dist and dist.get_backend() == 'nccl' else ', ranks share a GPU'})")
                   if world > 1 else "1 GPU",
                   "l2": "256 MiB flush before every timed step; working set (N x d_max x 16 B = 2 GiB) > L2"},
        "samples": st["samples"], "sketch_columns": st["sketch_columns"], "sketch_launches": sk_launches,
        "verified_error": verr,
        "verified_how": "16 Gaussian probes, all rows: ||H X - K X|| / ||K X|| with K X from libh2's FP64 DMMA dense "
                        "sketch (an independent kernel path)",
        "verified_error_torch": verr_t,
        "verified_torch_how": "the same probes on 256 sampled rows with K X from plain torch FP64 elementwise ops",
        "verified_error_2norm": None if p2 is None else p2[0],
        "verified_2norm_how": "PAPER.md L447: ||H - K||_2 / ||K||_2, each by 8 power iterations from 8 stream vectors (largest) "
                              "(h2_verify_2norm, K x by libh2's FP64 DMMA dense sketch); lower-bound estimates",
        "step_ms": [round(t, 2) for t in times],
        "host_wall_ms": [round(s["t_total_ms"], 2) for s in stats],
        "ranks": {str(t): [st["rank_min"][t], st["rank_max"][t], round(st["rank_mean"][t], 1)]
                  for t in st["rank_min"]},
        "rounds": st["rounds"],
        "phase_ms": {k: round(v, 3) for k, v in st["t_phase_ms"].items()},
        "entries_evaluated_per_s": (st["entries_D"] + st["entries_B"]) / (ms / 1e3),
        "sketch_entries_per_s": st["entries_sketch"] / (ms / 1e3),
        "gpu_launches": int(sum(s["launches"] for s in stats)),
        "roofline": {"bound": "alu", "kernel": "sketch_tc_kernel (FP64 K evaluation + tcgen05 kind::i8 contraction)",
                     "achieved": achieved, "peak": FP64_PIPE_TOPS, "unit": "TOP/s (FP64 pipe ops)",
                     "frac": achieved / FP64_PIPE_TOPS, "traffic": traffic,
                     "entries_per_s": entries_launch / (per_launch_ms * 1e-3),
                     "int8_tensor_tops": int8_ops, "int8_tensor_frac": int8_ops / INT8_DENSE_TOPS,
                     "per_launch_ms": per_launch_ms,
                     # the int8 UMMA stream and the FP64 pipe serialise on an SM (profiles/
                     # r2_sketch_serialization.md): the kernel's bound is the SUM of both times
                     "serialised_bound": {
                         "t_fp64_ms": entries_launch * F_EVAL / (FP64_PIPE_TOPS * 1e12) * 1e3,
                         "t_int8_ms": entries_launch * ncol_launch * slices * 2 / (INT8_MEASURED_TOPS * 1e12) * 1e3,
                         "frac": (entries_launch * F_EVAL / (FP64_PIPE_TOPS * 1e12)
                                  + entries_launch * ncol_launch * slices * 2 / (INT8_MEASURED_TOPS * 1e12))
                                 / (per_launch_ms * 1e-3),
                         "int8_peak_tops": INT8_MEASURED_TOPS},
                     "note": f"achieved = N^2 entries x {F_EVAL} FP64 ops (SASS) per launch / CUDA-event time of the "
                             "sketch phase per 160-column pass (speculative: columns beyond the converged d are computed, not used); peak = 148 SM x 64 FP64 lanes/clk x 1.965 GHz "
                             "(microbenchmarked DFMA 37.0 TF/s = 99.5 %); traffic = ncu dram bytes per launch"},
        "whole_build_roofline": whole_build_roofline(st, ms, n, rows_local, sk_launches, ncol_launch, slices),
        "clocks": clk,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    if world == 1 and not args.no_c3 and args.workload == "cov3d_256k":
        del H
        # the other BASELINE configs, driver-timed in the same run (one GPU): configs[2] (the
        # north-star size N = 2^21), configs[0], configs[3], configs[4]
        out["north_star_c3"] = time_workload(g, torch, stream, flush, "cov3d_2m")
        out["other_configs"] = {nm: time_workload(g, torch, stream, flush, nm, steps=3)
                                for nm in ("cov2d_1k", "ie3d_1m", "h2update_1m")}
    print(json.dumps(out), flush=True)


def time_workload(g, torch, stream, flush, name, steps=2):
    """Driver-timed extra line for another BASELINE config on ONE GPU (`value` stays configs[1]):
    build time (CUDA events, 1 warm-up + `steps` timed builds, L2 flushed), samples, per-phase
    times, construction-proper time, the sketch roofline, and a verified error:
      configs[0] cov2d_1k : K X by plain torch FP64 ops (torch_kx_rows), all rows;
      configs[2] cov3d_2m, configs[3] ie3d_1m : the same on 256 sampled rows of 16 probes;
      configs[4] h2update_1m : M X = A_H X + U (U^T X) with the base's H^2 matvec (the operator the
        update compresses; the base build is untimed set-up, like PAPER.md L479)."""
    from synth import WORKLOADS, lowrank_factor
    w = WORKLOADS[name]
    g._lib.lib.h2_cache_trim()
    torch.cuda.empty_cache()
    X = w["points"]()
    n = X.shape[0]
    t0 = time.perf_counter()
    T = g.Tree(X, w["leaf"], 0.7)
    tree_s = time.perf_counter() - t0
    kern = (w["kernel"], w["param"])
    opts = dict(adaptive=True, d_init=32, d_blk=32, d_max=w.get("d_max", 512), p_os=w.get("p_os", 10))
    extra = {}
    upd = None
    if "update_rank" in w:
        t0 = time.perf_counter()
        Hb = g.build(T, kern, w["tol"])
        torch.cuda.synchronize()
        extra["base_build_s_untimed"] = round(time.perf_counter() - t0, 2)
        upd = (Hb, torch.from_numpy(lowrank_factor(n, w["update_rank"])).cuda())
        opts["update"] = upd
    # warm-up builds: one, or four for configs[4] (near the 180 GB capacity the block cache
    # reaches its steady state -- ~7 cudaMalloc per build -- only after four builds; the first
    # ones spend 0.3-0.6 s re-mapping blocks, H2_TRACE=1, tools/c5_trace.py; serving oversized
    # free blocks instead ran out of memory)
    for _ in range(4 if upd is not None else 1):
        H = g.build(T, kern, w["tol"], **opts)
        del H
    times, stats = [], []
    for _ in range(steps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        H = g.build(T, kern, w["tol"], **opts)
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        stats.append(H.stats)
        if len(times) < steps:
            del H
    st = stats[-1]
    # libh2's block cache keeps the builds' freed workspaces; return them before torch allocates
    # the verification buffers (configs[4] runs at ~176 GB of the 180)
    g._lib.lib.h2_cache_trim()
    P = np.random.default_rng(2).standard_normal((n, 16))
    Pd = torch.from_numpy(P).cuda()
    HX = H.matvec(Pd).cpu().numpy()
    if upd is not None:
        MX = (upd[0].matvec(Pd) + upd[1] @ (upd[1].T @ Pd)).cpu().numpy()
        err, how = float(np.linalg.norm(HX - MX) / np.linalg.norm(MX)), "vs A_H X + U (U^T X), all rows"
    else:
        rows = np.arange(n) if n <= 4096 else np.sort(np.random.default_rng(9).choice(n, 256, replace=False))
        KX = torch_kx_rows(X[T.perm], w["kernel"], w["param"], Pd, rows)
        err = float(np.linalg.norm(HX[rows] - KX) / np.linalg.norm(KX))
        how = (f"vs K X from plain torch FP64 elementwise ops, {'all' if n <= 4096 else len(rows)} rows "
               "(16 Gaussian probes)")
    ms = float(np.mean(times))
    res = {"workload": name, "n": n, "tol": w["tol"], "build_s": ms / 1e3, "step_ms": [round(t, 1) for t in times],
           "samples": st["samples"], "verified_error": err, "verified_how": how,
           "phase_ms": {k: round(v, 1) for k, v in st["t_phase_ms"].items()},
           "construction_proper_ms": round(ms - st["t_phase_ms"]["sketch"], 1),
           "entries_evaluated_per_s": (st["entries_D"] + st["entries_B"]) / (ms / 1e3),
           "device_bytes": H.device_bytes(), "host_tree_s": round(tree_s, 2), "gpus": 1, **extra}
    if st["entries_sketch"] > 0 and upd is None:
        sk_launches = max(st["entries_sketch"] // (n * n), 1)
        per_launch = float(np.mean([s["t_phase_ms"]["sketch"] for s in stats])) / sk_launches
        f_eval = F_EVAL if w["kernel"] == "exp" else F_EVAL_HELM
        achieved = float(n) * n * f_eval / (per_launch * 1e-3) / 1e12
        res["sketch_roofline"] = {"bound": "alu", "achieved": achieved, "peak": FP64_PIPE_TOPS,
                                  "unit": "TOP/s (FP64 pipe ops)", "frac": achieved / FP64_PIPE_TOPS,
                                  "per_launch_ms": per_launch, "launches": int(sk_launches),
                                  "fp64_ops_per_entry": f_eval}
        exp = w["kernel"] == "exp"
        res["whole_build_roofline"] = whole_build_roofline(st, ms, n, n, int(sk_launches), 160 if exp else 128,
                                                           6 if exp else 7, f_eval)
    del H, T
    if upd is not None:
        del upd, opts
    g._lib.lib.h2_cache_trim()
    torch.cuda.empty_cache()
    return res


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    w = workload_cfg(args.workload)
    if args.impl == "reference":
        run_reference(args, w, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        ngpu = torch.cuda.device_count()
        if ngpu >= world:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            # fewer GPUs than ranks (functional check of the multi-rank path on one GPU):
            # ranks share the devices and the communicator stages through the host (gloo)
            local_rank %= ngpu
            torch.cuda.set_device(local_rank)
            dist.init_process_group("gloo")
    run_ours(args, w, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
