"""ctypes front end of the C oracle (oracle/c/h2oracle.c) -- TEST INFRASTRUCTURE ONLY.

The C oracle is Algorithm 1 (§III-A/B) in plain C with every floating-point
operation in the order stated in its header (DESIGN.md §3 "exact-order specification"): the
reference of libh2's exact-order mode (bitwise parity on the rational test kernel) and the timed
CPU baseline (OpenMP).  This module only marshals arrays (tree CSR in, export arrays out) and
compiles the library with gcc on first use; it shares no code with paper_2506_16759_b200/.
"""
import ctypes as C
import os
import subprocess

import numpy as np

from .h2 import H2Matrix

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(_HERE, "c", "h2oracle.c")
LIB = os.path.join(_HERE, "c", "libh2oracle.so")
MAXD = 64
KINDS = {"exp": 0, "helmholtz": 1, "rational": 2, "table": 3}


def build_library(force=False):
    """gcc -O3 -mavx2 -mfma -ffp-contract=off -fopenmp (no contraction: every fma in the source is
    explicit; vectorisation over sample columns keeps each element's operation order)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".{os.getpid()}.tmp"
        subprocess.run(["gcc", "-O3", "-mavx2", "-mfma", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC",
                        "-std=gnu11", "-o", tmp, SRC, "-lm"], check=True)
        os.replace(tmp, LIB)
    return LIB


class _Tree(C.Structure):
    _fields_ = [("n", C.c_int64), ("leaf_depth", C.c_int32), ("pts", C.c_void_p), ("begin", C.c_void_p),
                ("end", C.c_void_p), ("near_ptr", C.c_void_p), ("near_idx", C.c_void_p),
                ("far_ptr", C.c_void_p * MAXD), ("far_idx", C.c_void_p * MAXD)]


class _Opts(C.Structure):
    _fields_ = [("d_init", C.c_int32), ("d_blk", C.c_int32), ("d_max", C.c_int32), ("adaptive", C.c_int32),
                ("tol_rule", C.c_int32), ("tol_safety", C.c_double), ("norm", C.c_double),
                ("eps_decay", C.c_double), ("p_os", C.c_int32), ("max_rank", C.c_int32), ("seed", C.c_uint64),
                ("stream_id", C.c_uint32), ("threads", C.c_int32), ("omega_ext", C.c_void_p),
                ("ld_ext", C.c_int64), ("dense", C.c_void_p), ("ld_dense", C.c_int64), ("y_table", C.c_void_p),
                ("ld_table", C.c_int64), ("table_cols", C.c_int32)]


class _Result(C.Structure):
    _fields_ = [("status", C.c_int32), ("samples", C.c_int32), ("top", C.c_int32), ("leaf_depth", C.c_int32),
                ("failed_depth", C.c_int32), ("rounds", C.c_int32 * MAXD), ("eps", C.c_double),
                ("t_sketch", C.c_double), ("t_gen", C.c_double), ("t_bsr", C.c_double), ("t_cpqr", C.c_double),
                ("t_id", C.c_double), ("t_total", C.c_double),
                ("rank", C.POINTER(C.c_int32) * MAXD), ("skel", C.POINTER(C.c_int32) * MAXD),
                ("basis", C.POINTER(C.c_double) * MAXD), ("cert", C.POINTER(C.c_double) * MAXD),
                ("B", C.POINTER(C.c_double) * MAXD), ("nskel", C.c_int64 * MAXD), ("nbasis", C.c_int64 * MAXD),
                ("nB", C.c_int64 * MAXD), ("D", C.POINTER(C.c_double)), ("nD", C.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build_library())
        L.h2o_build.restype = C.POINTER(_Result)
        L.h2o_build.argtypes = [C.POINTER(_Tree), C.c_int32, C.c_double, C.c_double, C.POINTER(_Opts)]
        L.h2o_free.argtypes = [C.POINTER(_Result)]
        L.h2o_omega.argtypes = [C.c_uint64, C.c_uint32, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_void_p,
                                C.c_int64]
        L.h2o_philox4x32_10.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.h2o_cpqr.restype = C.c_int
        L.h2o_cpqr.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_double, C.c_int32, C.c_void_p, C.c_void_p]
        L.h2o_dense_sketch.argtypes = [C.c_int, C.c_double, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                                       C.c_int64, C.c_int32, C.c_void_p, C.c_int64]
        L.h2o_kernel_block.argtypes = [C.c_int, C.c_double, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                       C.c_void_p]
        L.h2o_max_threads.restype = C.c_int
        _lib = L
    return _lib


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def _csr(pairs, nrows):
    pairs = np.asarray(pairs, np.int64).reshape(-1, 2)
    order = np.lexsort((pairs[:, 1], pairs[:, 0]))
    pairs = pairs[order]
    ptr = np.zeros(nrows + 1, np.int64)
    np.add.at(ptr, pairs[:, 0] + 1, 1)
    return np.cumsum(ptr), np.ascontiguousarray(pairs[:, 1], dtype=np.int32)


class TreeArrays:
    """The oracle's tree (oracle.geometry) as flat arrays for the C oracle: tree-order points
    zero padded to 3D, heap-order cluster ranges, leaf near CSR, far CSR per depth."""

    def __init__(self, tree, part, points):
        X = np.asarray(points, np.float64)
        self.tree, self.part = tree, part
        self.n, Dl = tree.n, tree.leaf_depth
        self.pts = np.zeros((tree.n, 3))
        self.pts[:, :X.shape[1]] = X[tree.perm]
        self.begin = np.concatenate([np.asarray(tree.begin[t], np.int64) for t in range(Dl + 1)])
        self.end = np.concatenate([np.asarray(tree.end[t], np.int64) for t in range(Dl + 1)])
        self.near_ptr, self.near_idx = _csr(part.near, 1 << Dl)
        self.far = [_csr(part.far[t], 1 << t) if len(part.far[t]) else None for t in range(Dl + 1)]
        s = _Tree()
        s.n, s.leaf_depth = tree.n, Dl
        s.pts, s.begin, s.end = _p(self.pts), _p(self.begin), _p(self.end)
        s.near_ptr, s.near_idx = _p(self.near_ptr), _p(self.near_idx)
        for t in range(Dl + 1):
            if self.far[t] is not None:
                s.far_ptr[t], s.far_idx[t] = _p(self.far[t][0]), _p(self.far[t][1])
        self.struct = s


class NotConverged(RuntimeError):
    pass


class Result:
    """Export arrays of a C-oracle build in libh2's include/h2.h layouts (per depth t)."""

    def __init__(self, r, ta):
        self.samples, self.top, self.leaf_depth = r.samples, r.top, r.leaf_depth
        self.eps = r.eps
        self.rounds = {t: r.rounds[t] for t in range(r.top, r.leaf_depth + 1)}
        self.seconds = {"sketch": r.t_sketch, "gen": r.t_gen, "bsr": r.t_bsr, "cpqr": r.t_cpqr, "id": r.t_id,
                        "total": r.t_total}
        self.rank, self.skel, self.basis, self.cert, self.B = {}, {}, {}, {}, {}
        for t in range(r.top, r.leaf_depth + 1):
            nc = 1 << t
            self.rank[t] = np.ctypeslib.as_array(r.rank[t], (nc,)).copy()
            self.skel[t] = np.ctypeslib.as_array(r.skel[t], (max(r.nskel[t], 1),))[:r.nskel[t]].copy()
            self.basis[t] = np.ctypeslib.as_array(r.basis[t], (max(r.nbasis[t], 1),))[:r.nbasis[t]].copy()
            self.cert[t] = np.ctypeslib.as_array(r.cert[t], (2 * nc,)).copy().reshape(-1, 2)
            self.B[t] = np.ctypeslib.as_array(r.B[t], (max(r.nB[t], 1),))[:r.nB[t]].copy()
        self.D = np.ctypeslib.as_array(r.D, (max(r.nD, 1),))[:r.nD].copy()
        self._ta = ta

    def to_h2matrix(self):
        """The same H^2 as an oracle.h2.H2Matrix (for oracle.h2.matvec / to_dense)."""
        ta = self._ta
        tree, part, Dl = ta.tree, ta.part, self.leaf_depth
        H = H2Matrix(tree, part, self.top)
        H.samples, H.eps = self.samples, self.eps
        sz = lambda t, c: int(tree.end[t][c] - tree.begin[t][c])
        for t in range(self.top, Dl + 1):
            k = self.rank[t].astype(np.int64)
            H.rank[t] = k
            H.skel[t] = np.split(self.skel[t].astype(np.int64), np.cumsum(k)[:-1])
            m = [sz(t, c) for c in range(1 << t)] if t == Dl else \
                [int(self.rank[t + 1][2 * c] + self.rank[t + 1][2 * c + 1]) for c in range(1 << t)]
            X, o = [], 0
            for mi, ki in zip(m, k):
                X.append(self.basis[t][o:o + mi * ki].reshape(mi, ki))
                o += mi * ki
            H.X[t] = X
            blocks, o = {}, 0
            for (s, b) in part.far[t]:
                if s < b:
                    nb = k[s] * k[b]
                    blocks[(int(s), int(b))] = self.B[t][o:o + nb].reshape(k[s], k[b])
                    o += nb
            H.B[t] = {}
            for (s, b) in part.far[t]:
                s, b = int(s), int(b)
                H.B[t][(s, b)] = blocks[(s, b)] if s < b else blocks[(b, s)].T
        o, Dd = 0, {}
        for (s, b) in part.near:
            if s <= b:
                nb = sz(Dl, s) * sz(Dl, b)
                Dd[(int(s), int(b))] = self.D[o:o + nb].reshape(sz(Dl, s), sz(Dl, b))
                o += nb
        for (s, b) in part.near:
            s, b = int(s), int(b)
            H.D[(s, b)] = Dd[(s, b)] if s <= b else Dd[(b, s)].T
        return H


def build(ta: TreeArrays, kind, param, tol, d_init=32, d_blk=32, d_max=512, adaptive=True, tol_rule="rms",
          tol_safety=0.04, norm=0.0, eps_decay=1.25, p_os=10, max_rank=0, seed=1, stream_id=0, threads=0,
          omega_ext=None, dense=None, y_table=None):
    """Algorithm 1 in the C oracle.  Defaults = libh2's h2_build_opts_default (R9-R12,
    R31).  omega_ext: optional (n, >= d_max) float64 Omega (tree-order rows) instead of the
    Philox stream; kind "table" with dense = (n, n) tree-order operator.  Raises NotConverged at
    d_max (R26)."""
    o = _Opts()
    o.d_init, o.d_blk, o.d_max, o.adaptive = d_init, d_blk, d_max, int(bool(adaptive))
    o.tol_rule = 0 if tol_rule == "rms" else 1
    o.tol_safety, o.norm, o.eps_decay = tol_safety, norm, eps_decay
    o.p_os, o.max_rank = p_os, (max_rank or 0)
    o.seed, o.stream_id, o.threads = seed, stream_id, threads
    keep = None
    if omega_ext is not None:
        keep = np.ascontiguousarray(omega_ext, dtype=np.float64)
        o.omega_ext, o.ld_ext = keep.ctypes.data, keep.shape[1]
    keep3 = None
    if y_table is not None:   # the sketch supplied as a table (n, c): Y columns 0..c-1
        keep3 = np.ascontiguousarray(y_table, dtype=np.float64)
        o.y_table, o.ld_table, o.table_cols = keep3.ctypes.data, keep3.shape[1], keep3.shape[1]
    keep2 = None
    if dense is not None:
        keep2 = np.ascontiguousarray(dense, dtype=np.float64)
        o.dense, o.ld_dense = keep2.ctypes.data, keep2.shape[1]
    L = lib()
    rp = L.h2o_build(C.byref(ta.struct), KINDS[kind], float(param), float(tol), C.byref(o))
    r = rp.contents
    try:
        if r.status == -6:
            raise NotConverged(f"C oracle: d_max reached at depth {r.failed_depth}")
        if r.status == -2:
            raise ValueError(f"C oracle: the sketch table ran out of columns at depth {r.failed_depth}")
        if r.status != 0:
            raise ValueError(f"C oracle: status {r.status}")
        return Result(r, ta)
    finally:
        L.h2o_free(rp)


def omega(seed, stream, row0, nrows, col0, ncols):
    out = np.empty((nrows, ncols))
    lib().h2o_omega(seed, stream, row0, nrows, col0, ncols, _p(out), ncols)
    return out


def cpqr(A_rows, eps, kmax=0):
    """CPQR of the operand whose columns are the rows of A_rows (m x d): (k, perm, factored, cert)."""
    A = np.array(A_rows, dtype=np.float64, order="C", copy=True)
    m, d = A.shape
    perm = np.empty(m, np.int32)
    cert = np.empty(2)
    k = lib().h2o_cpqr(_p(A), m, d, float(eps), int(kmax), _p(perm), _p(cert))
    return k, perm.astype(np.int64), A, cert


def dense_sketch(ta: TreeArrays, kind, param, Om, rows=None):
    Om = np.ascontiguousarray(Om, np.float64)
    r0, r1 = (0, ta.n) if rows is None else rows
    Y = np.empty((r1 - r0, Om.shape[1]))
    lib().h2o_dense_sketch(KINDS[kind], float(param), _p(ta.pts), ta.n, r0, r1, _p(Om), Om.shape[1], Om.shape[1],
                           _p(Y), Om.shape[1])
    return Y


def kernel_block(ta: TreeArrays, kind, param, rows, cols):
    rows = np.ascontiguousarray(rows, np.int64)
    cols = np.ascontiguousarray(cols, np.int64)
    out = np.empty((len(rows), len(cols)))
    lib().h2o_kernel_block(KINDS[kind], float(param), _p(ta.pts), _p(rows), len(rows), _p(cols), len(cols), _p(out))
    return out


def max_threads():
    return int(lib().h2o_max_threads())
