"""Thin Python binding of libh2 (include/h2.h): argument marshalling only.

PyTorch provides device memory, streams and process groups; every step of Algorithm 1
 runs in the sm_100a kernels of libh2.so.  Names follow the paper:
``Tree`` (cluster tree + block partition, §II-A), ``build`` (Algorithm 1, returns an
``H2Matrix`` holding U, E, B, D and the skeletons I~), ``H2Matrix.matvec``.
"""
import ctypes as C

import numpy as np
import torch

from . import _lib as L
from ._lib import check, lib

KERNELS = {"exp": L.H2_K_EXP, "helmholtz": L.H2_K_HELMHOLTZ, "rational": L.H2_K_RATIONAL}


def _ptr(t):
    return C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class _CudaView:
    """__cuda_array_interface__ wrapper so torch can view a libh2-owned / callback buffer."""

    def __init__(self, ptr, shape, strides_elems, typestr="<f8", itemsize=8):
        self.__cuda_array_interface__ = {
            "shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False), "version": 3,
            "strides": tuple(s * itemsize for s in strides_elems)}


def device_view(ptr, shape, strides, dtype=torch.float64):
    typestr, size = {torch.float64: ("<f8", 8), torch.int32: ("<i4", 4), torch.int64: ("<i8", 8),
                     torch.uint8: ("|u1", 1)}[dtype]
    return torch.as_tensor(_CudaView(ptr, shape, strides, typestr, size), device="cuda")


class Tree:
    """KD-tree cluster tree + dual-traversal partition (§II-A; R1-R6).

    points: n x dim float64 in original order (host).  The tree keeps tree-ordered
    coordinates on the current CUDA device for the built-in kernels."""

    def __init__(self, points, leaf_size=64, eta=0.7, dist_rule="center", _handle=None, asynchronous=False):
        """asynchronous=True: h2_tree_build_async -- the block partition is built on a host thread
        and waited for by the first call that needs it; h2_build's first sketch pass overlaps it.
        The partition-dependent attributes below are then fetched on first access."""
        P = np.ascontiguousarray(points, dtype=np.float64)
        if P.ndim == 1:
            P = P[:, None]
        self.points = P
        self.n = P.shape[0]
        h = _handle
        if h is None:
            h = C.c_void_p()
            fn = lib.h2_tree_build_async if asynchronous else lib.h2_tree_build
            check(fn(P.ctypes.data_as(C.c_void_p), P.shape[0], P.shape[1], leaf_size, float(eta),
                     L.H2_DIST_CENTER if dist_rule == "center" else L.H2_DIST_BOX, C.byref(h)))
        self._h = h
        self._info = None
        self._near = self._far = None
        if not asynchronous:
            self._load_info()

    def _load_info(self):
        info = L.h2_tree_info()
        check(lib.h2_tree_get_info(self._h, C.byref(info)))
        nnodes = (1 << (info.leaf_depth + 1)) - 1
        perm = np.empty(self.n, np.int64)
        b = np.empty(nnodes, np.int64)
        e = np.empty(nnodes, np.int64)
        check(lib.h2_tree_export(self._h, perm.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p),
                                 e.ctypes.data_as(C.c_void_p), None))
        self._info = dict(dim=info.dim, leaf_size=info.leaf_size, leaf_depth=info.leaf_depth,
                          top_depth=info.top_depth, near_nnz=info.near_nnz, far_nnz_total=info.far_nnz_total,
                          csp=info.csp, perm=perm,
                          begin=[b[(1 << t) - 1:(1 << (t + 1)) - 1] for t in range(info.leaf_depth + 1)],
                          end=[e[(1 << t) - 1:(1 << (t + 1)) - 1] for t in range(info.leaf_depth + 1)])

    def __getattr__(self, name):   # partition-dependent attributes, loaded on first access
        if name in ("dim", "leaf_size", "leaf_depth", "top_depth", "near_nnz", "far_nnz_total", "csp", "perm",
                    "begin", "end"):
            if self.__dict__.get("_info") is None:
                self._load_info()
            return self.__dict__["_info"][name]
        raise AttributeError(name)

    @classmethod
    def from_partition(cls, points, perm, begin, end, near, far):
        """A partition built elsewhere (h2_tree_import): perm (tree -> original index), begin/end
        per depth (lists of int arrays, depth 0 = root), near (ordered leaf pairs, k x 2), far
        (per depth, ordered admissible pairs, k_t x 2)."""
        P = np.ascontiguousarray(points, dtype=np.float64)
        if P.ndim == 1:
            P = P[:, None]
        Dl = len(begin) - 1
        perm = np.ascontiguousarray(perm, np.int64)
        b = np.ascontiguousarray(np.concatenate([np.asarray(x, np.int64) for x in begin]))
        e = np.ascontiguousarray(np.concatenate([np.asarray(x, np.int64) for x in end]))
        nr = np.ascontiguousarray(np.asarray(near, np.int32).reshape(-1, 2))
        fr = [np.ascontiguousarray(np.asarray(f, np.int32).reshape(-1, 2)) for f in far]
        fnnz = np.array([len(f) for f in fr], np.int64)
        fptr = (C.c_void_p * (Dl + 1))(*[f.ctypes.data if len(f) else None for f in fr])
        d = L.h2_tree_desc(P.shape[0], P.shape[1], Dl, P.ctypes.data, perm.ctypes.data, b.ctypes.data,
                           e.ctypes.data, len(nr), nr.ctypes.data, fnnz.ctypes.data, C.cast(fptr, C.c_void_p))
        h = C.c_void_p()
        check(lib.h2_tree_import(C.byref(d), C.byref(h)))
        return cls(P, _handle=h)

    @property
    def near(self):
        """Ordered near pairs (s, b) of the leaf depth (exported on first use)."""
        if self._near is None:
            near = np.empty((self.near_nnz, 2), np.int32)
            check(lib.h2_tree_export(self._h, None, None, None, near.ctypes.data_as(C.c_void_p)))
            self._near = near.astype(np.int64)
        return self._near

    @property
    def far(self):
        """Per depth: ordered admissible pairs (s, b) (exported on first use)."""
        if self._far is None:
            far = []
            for t in range(self.leaf_depth + 1):
                cnt = C.c_int64()
                check(lib.h2_tree_far_count(self._h, t, C.byref(cnt)))
                f = np.empty((cnt.value, 2), np.int32)
                if cnt.value:
                    check(lib.h2_tree_export_far(self._h, t, f.ctypes.data_as(C.c_void_p)))
                far.append(f.astype(np.int64))
            self._far = far
        return self._far

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.h2_tree_free(h)
            self._h = None


def build_opts(**kw):
    o = L.h2_build_opts()
    lib.h2_build_opts_default(C.byref(o))
    names = {"tol_rule": None}
    for k, v in kw.items():
        if v is None:
            continue
        if k == "tol_rule":
            v = {"rms": L.H2_TOL_RMS, "literal": L.H2_TOL_LITERAL}[v] if isinstance(v, str) else v
        if k == "sketch_split":
            v = {"rows": L.H2_SPLIT_ROWS, "cols": L.H2_SPLIT_COLS}[v] if isinstance(v, str) else v
        if k == "adaptive":
            v = int(bool(v))
        if not hasattr(o, k) and k not in names:
            raise TypeError(f"unknown build option {k}")
        setattr(o, k, v)
    return o


def _kernel(kind, param):
    return L.h2_kernel(KERNELS[kind], float(param))


class H2Matrix:
    """Result of Algorithm 1: U (leaves), E (transfer), B (couplings), D (dense), I~ (skeletons)."""

    def __init__(self, handle, tree, stats, keep=(), nonsym=False):
        self._h = handle
        self.nonsym = nonsym      # h2_build_nonsym: row side (rank/skel/basis) + column side (*_c)
        self.tree = tree          # the matrix references the tree: keep it alive
        self.stats = stats
        self._keep = keep

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.h2_free(h)
            self._h = None

    # ---- inspection (copies to host numpy)
    def _export(self, what, depth=0, dtype=np.float64):
        cnt = C.c_int64()
        check(lib.h2_export_size(self._h, what, depth, C.byref(cnt)))
        out = np.empty(cnt.value, dtype)
        if cnt.value:
            check(lib.h2_export(self._h, what, depth, out.ctypes.data_as(C.c_void_p)))
        return out

    @property
    def top_depth(self):
        return self.stats["top_depth"]

    @property
    def samples(self):
        return self.stats["samples"]

    def rank(self, t, side=0):
        """side 0: row ranks (the symmetric build's only side); 1: column ranks (non-symmetric)."""
        return self._export(L.H2_X_RANK_C if side else L.H2_X_RANK, t, np.int32).astype(np.int64)

    def ranks_and_skeletons(self, side=0):
        """Ranks and skeleton indices of every processed depth (top..leaf, concatenated) in two
        calls (h2_export with H2_ALL_DEPTHS): the end-to-end result read."""
        rk = self._export(L.H2_X_RANK_C if side else L.H2_X_RANK, L.H2_ALL_DEPTHS, np.int32)
        sk = self._export(L.H2_X_SKEL_C if side else L.H2_X_SKEL, L.H2_ALL_DEPTHS, np.int32)
        return rk, sk

    def skel(self, t, side=0):
        r = self.rank(t, side)
        s = self._export(L.H2_X_SKEL_C if side else L.H2_X_SKEL, t, np.int32).astype(np.int64)
        return np.split(s, np.cumsum(r)[:-1])

    def panel_rows(self, t, side=0):
        if t == self.tree.leaf_depth:
            return (self.tree.end[t] - self.tree.begin[t]).astype(np.int64)
        rc = self.rank(t + 1, side)
        return rc[0::2] + rc[1::2]

    def basis(self, t, side=0):
        """X_tau per cluster of depth t (m x k): U_tau at the leaves, [E_nu1; E_nu2] above
        (side 1: the column bases V / [F1; F2] of a non-symmetric matrix)."""
        r = self.rank(t, side)
        m = self.panel_rows(t, side)
        x = self._export(L.H2_X_BASIS_C if side else L.H2_X_BASIS, t)
        out, o = [], 0
        for mi, ki in zip(m, r):
            out.append(x[o:o + mi * ki].reshape(mi, ki))
            o += mi * ki
        return out

    def cert(self, t, side=0):
        return self._export(L.H2_X_CERT_C if side else L.H2_X_CERT, t).reshape(-1, 2)

    def D_blocks(self):
        """dict (s, b) -> m_s x m_b for unique near pairs s <= b (every ordered pair if nonsym)."""
        Dl = self.tree.leaf_depth
        raw = self._export(L.H2_X_D)
        sz = self.tree.end[Dl] - self.tree.begin[Dl]
        out, o = {}, 0
        for s, b in self.tree.near:
            if s <= b or self.nonsym:
                n = sz[s] * sz[b]
                out[(int(s), int(b))] = raw[o:o + n].reshape(sz[s], sz[b])
                o += n
        return out

    def B_blocks(self, t):
        """dict (s, b) -> k_s x k_b for unique far pairs s < b of depth t (nonsym: every ordered
        pair, k_s x kc_b)."""
        r = self.rank(t)
        rc = self.rank(t, 1) if self.nonsym else r
        raw = self._export(L.H2_X_B, t)
        out, o = {}, 0
        for s, b in self.tree.far[t]:
            if s < b or self.nonsym:
                n = r[s] * rc[b]
                out[(int(s), int(b))] = raw[o:o + n].reshape(r[s], rc[b])
                o += n
        return out

    def verify(self, kernel=("exp", 0.2), q=8, seed=1, stream_id=2, dense=None, stream=None):
        """A-posteriori estimate (h2_verify): ||H Om_h - K Om_h||_F / ||K Om_h||_F
        over q held-out columns of the Omega stream (seed, stream_id); K the built-in kernel or
        the dense tree-order operator ``dense``."""
        sk = L.h2_sketch()
        sk.kern = _kernel(*kernel)
        if dense is not None:
            sk.kind, sk.A, sk.ld_A = L.H2_S_DENSE_MATRIX, dense.data_ptr(), dense.stride(0)
        else:
            sk.kind = L.H2_S_DENSE_KERNEL
        e = C.c_double()
        check(lib.h2_verify(self._h, C.byref(sk), q, seed, stream_id, _stream(stream), C.byref(e)))
        return e.value

    def verify_2norm(self, kernel=("exp", 0.2), iters=10, nvec=1, seed=1, stream_id=4, dense=None, stream=None):
        """The paper's error measure (h2_verify_2norm): (||H - K||_2 / ||K||_2,
        ||H - K||_2, ||K||_2), each 2-norm by ``iters`` power iterations from columns 0..nvec-1 of
        the Omega stream (seed, stream_id), the largest estimate; K the built-in kernel or the dense
        tree-order operator ``dense``."""
        sk = L.h2_sketch()
        sk.kern = _kernel(*kernel)
        if dense is not None:
            sk.kind, sk.A, sk.ld_A = L.H2_S_DENSE_MATRIX, dense.data_ptr(), dense.stride(0)
        else:
            sk.kind = L.H2_S_DENSE_KERNEL
        r, e, k = C.c_double(), C.c_double(), C.c_double()
        check(lib.h2_verify_2norm(self._h, C.byref(sk), iters, nvec, seed, stream_id, _stream(stream), C.byref(r),
                                  C.byref(e), C.byref(k)))
        return r.value, e.value, k.value

    def allgather(self, comm, stream=None):
        """Complete a distributed build on every rank (h2_matrix_allgather; collective)."""
        check(lib.h2_matrix_allgather(self._h, C.byref(comm.struct), _stream(stream)))
        return self

    def device_bytes(self):
        return int(lib.h2_matrix_device_bytes(self._h))

    # ---- H^2 matvec (tree-order rows)
    def matvec(self, x, alpha=1.0, beta=0.0, y=None, stream=None):
        """y = alpha K_H x + beta y for x: (n, q) float64 CUDA tensor (q <= 64)."""
        vec = x.dim() == 1
        X = x.reshape(x.shape[0], -1).contiguous()
        assert X.is_cuda and X.dtype == torch.float64 and X.shape[0] == self.tree.n
        q = X.shape[1]
        if y is None:
            y = torch.zeros_like(X)
            beta = 0.0
        check(lib.h2_matvec(self._h, _ptr(X), X.stride(0), _ptr(y), y.stride(0), q, float(alpha), float(beta),
                            _stream(stream)))
        return y[:, 0] if vec else y


def _stats_dict(s):
    d = {k: getattr(s, k) for k in ("samples", "failed_depth", "top_depth", "leaf_depth", "eps", "entries_D",
                                    "entries_B", "entries_sketch", "sketch_columns", "bytes_U", "bytes_E", "bytes_B", "bytes_D",
                                    "launches", "t_total_ms", "verify_error", "verify_rebuilds", "tol_safety_used",
                                    "cpqr_variants", "norm_est")}
    lo, hi = s.top_depth, s.leaf_depth
    d["rounds"] = {t: s.rounds[t] for t in range(lo, hi + 1)}
    d["rank_min"] = {t: s.rank_min[t] for t in range(lo, hi + 1)}
    d["rank_max"] = {t: s.rank_max[t] for t in range(lo, hi + 1)}
    d["rank_mean"] = {t: s.rank_mean[t] for t in range(lo, hi + 1)}
    d["t_phase_ms"] = {L.PHASES[i]: s.t_phase_ms[i] for i in range(L.H2_NPHASE)}
    d["t_depth_ms"] = {t: s.t_depth_ms[t] for t in range(lo, hi + 1)}
    d["work_flops"] = {L.PHASES[i]: s.work_flops[i] for i in range(L.H2_NPHASE)}
    d["work_bytes"] = {L.PHASES[i]: s.work_bytes[i] for i in range(L.H2_NPHASE)}
    return d


def build(tree: Tree, kernel=("exp", 0.2), tol=1e-6, sketch=None, entry=None, stream=None, update=None, comm=None,
          h2_sketch=None, dense=None, nonsym=False, omega=None, **opts):
    """Algorithm 1 on the current device.

    kernel: (kind, param) built-in kernel used for the entry evaluator (and the dense sketch
    unless ``sketch`` is given).  sketch: optional callable sketch(omega, y, col0, row_begin,
    row_end) filling y (tree-order rows) for a black-box K_blk; entry: optional callable
    entry(row_idx, col_idx, blocks) (see include/h2.h h2_block_batch).  update=(H_base, U) or
    (H_base, U, V) (M = A_H + U V^T, with nonsym=True):
    recompress M = H_base + U U^T (H_base built on this tree, U a (n, r) float64
    CUDA tensor in tree order) with the library's H^2-matvec + low-rank sketch and entry
    extraction.  h2_sketch=H_base: the O(N) black-box sketch Y = A_H Omega of an existing H^2 on
    this tree (e.g. K at a tighter tolerance), entries from ``kernel``.
    dense=A: an explicit (n, n) float64 CUDA operator in TREE order (row-major): sketch A Omega
    (one DGEMM per draw) and entries A[i, j] (S§8(f) NEXT #4, a frontal-matrix stand-in).
    nonsym=True: the non-symmetric construction K ~ D + U B V^T (h2_build_nonsym; row bases from
    K Omega, column bases from K^T Psi); a ``sketch`` callable then receives transpose=0/1 as a
    keyword and must write K^T omega for transpose=1; ``dense`` A is used as given (A^T via DGEMM).
    comm: optional ``dist.Comm`` (one process per GPU): the construction is sharded
    by subtrees (h2_build_dist); call ``H.allgather(comm)`` before matvec / block export.
    omega: optional (n, >= d_max) float64 CUDA tensor, tree-order rows: an external Omega
    (h2_build_opts.omega_ext) instead of the h2_omega stream.
    opts: h2_build_opts fields (d_init, d_blk, d_max, adaptive, tol_rule,
    tol_safety, p_os, norm, max_rank, seed, stream_id, exact_order, norm_iters, eps_decay,
    sketch_split: "rows" | "cols" -- with comm and a ``sketch`` callable, "cols" calls it on this
    rank's slice of the sample columns for ALL rows and all-to-alls the slices into row shards)."""
    o = build_opts(**opts)
    kern = _kernel(*kernel)
    keep = []
    if omega is not None:
        assert omega.is_cuda and omega.dtype == torch.float64 and omega.shape[0] == tree.n and omega.stride(1) == 1
        keep.append(omega)
        o.omega_ext, o.ld_omega_ext = omega.data_ptr(), omega.stride(0)
    sk = L.h2_sketch()
    sk.kern = kern
    V = None
    if update is not None:
        Hb, U = update[0], update[1]
        V = update[2] if len(update) > 2 else None
        assert Hb.tree is tree, "update: the base H^2 must be built on the same Tree"
        U = U.contiguous()
        assert U.is_cuda and U.dtype == torch.float64 and U.shape[0] == tree.n
        keep += [Hb, U]
        sk.kind = L.H2_S_H2_LOWRANK
        sk.base, sk.U, sk.ld_U, sk.rank = Hb._h, U.data_ptr(), U.stride(0), U.shape[1]
        if V is not None:   # M = A_H + U V^T (non-symmetric: nonsym=True)
            V = V.contiguous()
            assert V.is_cuda and V.dtype == torch.float64 and V.shape == U.shape
            keep.append(V)
            sk.V, sk.ld_V = V.data_ptr(), V.stride(0)
    elif dense is not None:
        assert dense.is_cuda and dense.dtype == torch.float64 and dense.shape == (tree.n, tree.n)
        assert dense.stride(1) == 1
        keep.append(dense)
        sk.kind = L.H2_S_DENSE_MATRIX
        sk.A, sk.ld_A = dense.data_ptr(), dense.stride(0)
    elif h2_sketch is not None:
        assert h2_sketch.tree is tree, "h2_sketch: the H^2 must be built on the same Tree"
        keep.append(h2_sketch)
        sk.kind = L.H2_S_H2_LOWRANK
        sk.base, sk.U, sk.ld_U, sk.rank = h2_sketch._h, None, 0, 0
    elif sketch is None:
        sk.kind = L.H2_S_DENSE_KERNEL
    else:
        sk.kind = L.H2_S_CALLBACK

        def _sk(ctx, req):
            try:
                r = req.contents
                n, nr, nc = r.n, r.row_end - r.row_begin, r.ncols
                # the callback's torch work is enqueued on libh2's stream (req.stream): ordered
                # after the Omega generation and before the library's next kernels (h2.h)
                with torch.cuda.stream(torch.cuda.ExternalStream(r.stream or 0)):
                    om = device_view(r.omega, (n, nc), (r.ld_omega, 1))
                    y = device_view(r.y, (nr, nc), (r.ld_y, 1))
                    if nonsym:
                        sketch(om, y, r.col0, r.row_begin, r.row_end, transpose=r.transpose)
                    else:
                        sketch(om, y, r.col0, r.row_begin, r.row_end)
                return 0
            except Exception as exc:  # reported as H2_ERR_CALLBACK
                import traceback
                traceback.print_exc()
                return 1
        cb = L.SKETCH_FN(_sk)
        keep.append(cb)
        sk.fn = cb
    en = L.h2_entry()
    en.kern = kern
    if dense is not None:
        en.kind = L.H2_E_DENSE_MATRIX
        en.A, en.ld_A = dense.data_ptr(), dense.stride(0)
    elif update is not None:
        en.kind = L.H2_E_H2_LOWRANK
        en.base, en.U, en.ld_U, en.rank = sk.base, sk.U, sk.ld_U, sk.rank
        en.V, en.ld_V = sk.V, sk.ld_V
    elif entry is None:
        en.kind = L.H2_E_BUILTIN
    else:
        en.kind = L.H2_E_CALLBACK

        def _en(ctx, batch):
            try:
                b = batch.contents
                with torch.cuda.stream(torch.cuda.ExternalStream(b.stream or 0)):
                    entry(b)
                return 0
            except Exception:
                import traceback
                traceback.print_exc()
                return 1
        cb2 = L.ENTRY_FN(_en)
        keep.append(cb2)
        en.fn = cb2
    h = C.c_void_p()
    st = L.h2_build_stats()
    cm = None
    if nonsym:
        if comm is not None:   # sharded non-symmetric construction (h2_build_nonsym_dist)
            keep.append(comm)
            check(lib.h2_build_nonsym_dist(tree.handle, C.byref(sk), C.byref(en), float(tol), C.byref(o),
                                           C.byref(comm.struct), _stream(stream), C.byref(h), C.byref(st)))
        else:
            check(lib.h2_build_nonsym(tree.handle, C.byref(sk), C.byref(en), float(tol), C.byref(o),
                                      _stream(stream), C.byref(h), C.byref(st)))
        return H2Matrix(h, tree, _stats_dict(st), keep, nonsym=True)
    if comm is not None:
        cm = C.byref(comm.struct)
        keep.append(comm)
    check(lib.h2_build_dist(tree.handle, C.byref(sk), C.byref(en), float(tol), C.byref(o), cm, _stream(stream),
                            C.byref(h), C.byref(st)))
    return H2Matrix(h, tree, _stats_dict(st), keep)


def dense_sketch(tree: Tree, omega, kernel=("exp", 0.2), row_begin=0, row_end=None, out=None, stream=None,
                 omega_quarters=False):
    """Y(rows, :) = K(rows, :) Omega with the built-in kernel.  omega_quarters=True asserts that
    Omega is the h2 stream (entries q/4, |q| <= 32): the exp kernel then runs on the int8 tensor
    cores (exact); otherwise the FP64 DMMA kernel."""
    row_end = tree.n if row_end is None else row_end
    assert omega.is_cuda and omega.dtype == torch.float64 and omega.shape[0] == tree.n
    nc = omega.shape[1]
    if out is None:
        out = torch.empty((row_end - row_begin, nc), dtype=torch.float64, device=omega.device)
    check(lib.h2_dense_sketch(tree.handle, _kernel(*kernel), row_begin, row_end, _ptr(omega), omega.stride(0), nc,
                              _ptr(out), out.stride(0), L.H2_SKETCH_OMEGA_QUARTERS if omega_quarters else 0,
                              _stream(stream)))
    return out


def dense_op_sketch(A, omega, row_begin=0, row_end=None, out=None, stream=None, omega_quarters=False):
    """Y(rows, :) = A(rows, :) Omega for an explicit (n, n) float64 CUDA operator A (row-major):
    omega_quarters=True (Omega = the h2 stream) runs the int8 tensor-core product, else DGEMM."""
    n = A.shape[0]
    row_end = n if row_end is None else row_end
    assert A.is_cuda and A.dtype == torch.float64 and A.shape == (n, n) and A.stride(1) == 1
    assert omega.is_cuda and omega.dtype == torch.float64 and omega.shape[0] == n and omega.stride(1) == 1
    nc = omega.shape[1]
    if out is None:
        out = torch.empty((row_end - row_begin, nc), dtype=torch.float64, device=omega.device)
    check(lib.h2_dense_op_sketch(_ptr(A), A.stride(0), n, row_begin, row_end, _ptr(omega), omega.stride(0), nc,
                                 _ptr(out), out.stride(0), L.H2_SKETCH_OMEGA_QUARTERS if omega_quarters else 0,
                                 _stream(stream)))
    return out


def omega(nrows, ncols, seed=1, stream_id=0, row0=0, col0=0, device="cuda", stream=None):
    """Rows [row0,row0+nrows) x columns [col0,col0+ncols) of the Omega stream (Philox4x32-10)."""
    out = torch.empty((nrows, ncols), dtype=torch.float64, device=device)
    check(lib.h2_omega(seed, stream_id, row0, nrows, col0, ncols, _ptr(out), out.stride(0), _stream(stream)))
    return out
