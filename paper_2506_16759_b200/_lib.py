"""ctypes mirror of include/h2.h (argument marshalling only; all arithmetic runs in libh2.so).

The shared library is built in-tree (``paper_2506_16759_b200/libh2.so``) by
``__graft_entry__.build()`` / ``make -C paper_2506_16759_b200/csrc``.  There is no fallback:
importing this module without the library raises ImportError.
"""
import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("H2_LIB_PATH") or os.path.join(_HERE, "libh2.so")   # H2_LIB_PATH: a profiling build

H2_OK, H2_ERR_INVALID_ARG, H2_ERR_OOM, H2_ERR_CUDA, H2_ERR_NCCL = 0, -1, -2, -3, -4
H2_ERR_CALLBACK, H2_ERR_NOT_CONVERGED, H2_ERR_NONFINITE = -5, -6, -7
H2_DIST_CENTER, H2_DIST_BOX = 0, 1
H2_K_EXP, H2_K_HELMHOLTZ, H2_K_RATIONAL = 0, 1, 2
H2_S_DENSE_KERNEL, H2_S_CALLBACK, H2_S_H2_LOWRANK, H2_S_DENSE_MATRIX = 0, 1, 2, 3
H2_E_BUILTIN, H2_E_CALLBACK, H2_E_H2_LOWRANK, H2_E_DENSE_MATRIX = 0, 1, 2, 3
H2_TOL_RMS, H2_TOL_LITERAL = 0, 1
H2_SPLIT_ROWS, H2_SPLIT_COLS = 0, 1
H2_X_RANK, H2_X_SKEL, H2_X_BASIS, H2_X_D, H2_X_B, H2_X_CERT, H2_X_RANK_C, H2_X_SKEL_C, H2_X_BASIS_C, H2_X_CERT_C = range(10)
H2_SKETCH_OMEGA_QUARTERS = 1
H2_CQ_V_WARP, H2_CQ_V_SMEM, H2_CQ_V_GLOBAL, H2_CQ_V_EXACT, H2_CQ_V_CLUSTER = 1, 2, 4, 8, 16
PHASES = ["rand", "sketch", "gen", "bsr", "cpqr", "id", "misc"]
H2_ALL_DEPTHS = -1   # h2_export: every processed depth concatenated (ranks / skeletons)
H2_NPHASE = len(PHASES)


class h2_tree_info(C.Structure):
    _fields_ = [("n", C.c_int64), ("dim", C.c_int32), ("leaf_size", C.c_int32), ("leaf_depth", C.c_int32),
                ("top_depth", C.c_int32), ("near_nnz", C.c_int64), ("far_nnz_total", C.c_int64),
                ("csp", C.c_int32)]


class h2_tree_desc(C.Structure):
    _fields_ = [("n", C.c_int64), ("dim", C.c_int32), ("leaf_depth", C.c_int32), ("coords", C.c_void_p),
                ("perm", C.c_void_p), ("begin", C.c_void_p), ("end", C.c_void_p), ("near_nnz", C.c_int64),
                ("near_pairs", C.c_void_p), ("far_nnz", C.c_void_p), ("far_pairs", C.c_void_p)]


class h2_kernel(C.Structure):
    _fields_ = [("kind", C.c_int32), ("param", C.c_double)]


class h2_sketch_req(C.Structure):
    _fields_ = [("n", C.c_int64), ("row_begin", C.c_int64), ("row_end", C.c_int64), ("col0", C.c_int32),
                ("ncols", C.c_int32), ("omega", C.c_void_p), ("ld_omega", C.c_int64), ("y", C.c_void_p),
                ("ld_y", C.c_int64), ("stream", C.c_void_p), ("transpose", C.c_int32)]


SKETCH_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(h2_sketch_req))


class h2_sketch(C.Structure):
    _fields_ = [("kind", C.c_int32), ("kern", h2_kernel), ("fn", SKETCH_FN), ("ctx", C.c_void_p),
                ("base", C.c_void_p), ("U", C.c_void_p), ("ld_U", C.c_int64), ("rank", C.c_int32),
                ("A", C.c_void_p), ("ld_A", C.c_int64), ("V", C.c_void_p), ("ld_V", C.c_int64)]


class h2_block_batch(C.Structure):
    _fields_ = [("nblocks", C.c_int64), ("m", C.c_void_p), ("nc", C.c_void_p), ("row_off", C.c_void_p),
                ("col_off", C.c_void_p), ("row_idx", C.c_void_p), ("col_idx", C.c_void_p), ("out", C.c_void_p),
                ("ld", C.c_void_p), ("stream", C.c_void_p)]


ENTRY_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(h2_block_batch))


class h2_entry(C.Structure):
    _fields_ = [("kind", C.c_int32), ("kern", h2_kernel), ("fn", ENTRY_FN), ("ctx", C.c_void_p),
                ("base", C.c_void_p), ("U", C.c_void_p), ("ld_U", C.c_int64), ("rank", C.c_int32),
                ("A", C.c_void_p), ("ld_A", C.c_int64), ("V", C.c_void_p), ("ld_V", C.c_int64)]


class h2_build_opts(C.Structure):
    _fields_ = [("d_init", C.c_int32), ("d_blk", C.c_int32), ("d_max", C.c_int32), ("adaptive", C.c_int32),
                ("tol_rule", C.c_int32), ("tol_safety", C.c_double), ("p_os", C.c_int32), ("norm", C.c_double),
                ("max_rank", C.c_int32), ("seed", C.c_uint64), ("stream_id", C.c_uint32),
                ("verify_probes", C.c_int32), ("verify_retries", C.c_int32), ("eps_decay", C.c_double),
                ("exact_order", C.c_int32), ("omega_ext", C.c_void_p), ("ld_omega_ext", C.c_int64),
                ("norm_iters", C.c_int32), ("sketch_split", C.c_int32)]


class h2_build_stats(C.Structure):
    _fields_ = [("samples", C.c_int32), ("failed_depth", C.c_int32), ("top_depth", C.c_int32),
                ("leaf_depth", C.c_int32), ("rounds", C.c_int32 * 64), ("rank_min", C.c_int32 * 64),
                ("rank_max", C.c_int32 * 64), ("rank_mean", C.c_double * 64), ("eps", C.c_double),
                ("entries_D", C.c_int64), ("entries_B", C.c_int64), ("entries_sketch", C.c_int64),
                ("sketch_columns", C.c_int64),
                ("bytes_U", C.c_int64), ("bytes_E", C.c_int64), ("bytes_B", C.c_int64), ("bytes_D", C.c_int64),
                ("launches", C.c_int64), ("t_phase_ms", C.c_double * H2_NPHASE), ("t_total_ms", C.c_double),
                ("verify_error", C.c_double), ("verify_rebuilds", C.c_int32), ("tol_safety_used", C.c_double),
                ("cpqr_variants", C.c_int32), ("t_depth_ms", C.c_double * 64), ("norm_est", C.c_double),
                ("work_flops", C.c_double * H2_NPHASE), ("work_bytes", C.c_double * H2_NPHASE)]


ALLGATHERV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_void_p)
ALLTOALLV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_void_p,
                           C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_void_p)


class h2_comm(C.Structure):
    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32), ("allgatherv", ALLGATHERV_FN), ("ctx", C.c_void_p),
                ("nccl", C.c_void_p), ("alltoallv", ALLTOALLV_FN)]


# every symbol include/h2.h declares, with its ctypes signature
_P = C.c_void_p
SIGNATURES = {
    "h2_tree_build": (C.c_int, [_P, C.c_int64, C.c_int32, C.c_int32, C.c_double, C.c_int32, C.POINTER(_P)]),
    "h2_tree_build_async": (C.c_int, [_P, C.c_int64, C.c_int32, C.c_int32, C.c_double, C.c_int32, C.POINTER(_P)]),
    "h2_tree_import": (C.c_int, [C.POINTER(h2_tree_desc), C.POINTER(_P)]),
    "h2_tree_get_info": (C.c_int, [_P, C.POINTER(h2_tree_info)]),
    "h2_tree_export": (C.c_int, [_P, _P, _P, _P, _P]),
    "h2_tree_far_count": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_int64)]),
    "h2_tree_export_far": (C.c_int, [_P, C.c_int32, _P]),
    "h2_tree_free": (None, [_P]),
    "h2_build_opts_default": (None, [C.POINTER(h2_build_opts)]),
    "h2_build": (C.c_int, [_P, C.POINTER(h2_sketch), C.POINTER(h2_entry), C.c_double, C.POINTER(h2_build_opts), _P,
                           C.POINTER(_P), C.POINTER(h2_build_stats)]),
    "h2_build_nonsym": (C.c_int, [_P, C.POINTER(h2_sketch), C.POINTER(h2_entry), C.c_double,
                                  C.POINTER(h2_build_opts), _P, C.POINTER(_P), C.POINTER(h2_build_stats)]),
    "h2_build_nonsym_dist": (C.c_int, [_P, C.POINTER(h2_sketch), C.POINTER(h2_entry), C.c_double,
                                       C.POINTER(h2_build_opts), C.POINTER(h2_comm), _P, C.POINTER(_P),
                                       C.POINTER(h2_build_stats)]),
    "h2_cache_bytes": (C.c_int64, []),
    "h2_cache_trim": (None, []),
    "h2_verify": (C.c_int, [_P, C.POINTER(h2_sketch), C.c_int32, C.c_uint64, C.c_uint32, _P, C.POINTER(C.c_double)]),
    "h2_verify_2norm": (C.c_int, [_P, C.POINTER(h2_sketch), C.c_int32, C.c_int32, C.c_uint64, C.c_uint32, _P,
                                  C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "h2_build_dist": (C.c_int, [_P, C.POINTER(h2_sketch), C.POINTER(h2_entry), C.c_double, C.POINTER(h2_build_opts),
                                C.POINTER(h2_comm), _P, C.POINTER(_P), C.POINTER(h2_build_stats)]),
    "h2_matrix_allgather": (C.c_int, [_P, C.POINTER(h2_comm), _P]),
    "h2_comm_get_unique_id": (C.c_int, [_P]),
    "h2_comm_init": (C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(C.POINTER(h2_comm))]),
    "h2_comm_free": (None, [C.POINTER(h2_comm)]),
    "h2_comm_allgatherv": (C.c_int, [C.POINTER(h2_comm), _P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), _P]),
    "h2_comm_alltoallv": (C.c_int, [C.POINTER(h2_comm), _P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), _P,
                                    C.POINTER(C.c_int64), C.POINTER(C.c_int64), _P]),
    "h2_dist_range": (C.c_int, [C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "h2_matvec": (C.c_int, [_P, _P, C.c_int64, _P, C.c_int64, C.c_int32, C.c_double, C.c_double, _P]),
    "h2_dense_sketch": (C.c_int, [_P, h2_kernel, C.c_int64, C.c_int64, _P, C.c_int64, C.c_int32, _P, C.c_int64,
                                  C.c_int32, _P]),
    "h2_dense_op_sketch": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int64, C.c_int64, _P, C.c_int64, C.c_int32, _P,
                                     C.c_int64, C.c_int32, _P]),
    "h2_omega": (C.c_int, [C.c_uint64, C.c_uint32, C.c_int64, C.c_int64, C.c_int32, C.c_int32, _P, C.c_int64, _P]),
    "h2_export_size": (C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(C.c_int64)]),
    "h2_export": (C.c_int, [_P, C.c_int32, C.c_int32, _P]),
    "h2_matrix_get_stats": (C.c_int, [_P, C.POINTER(h2_build_stats)]),
    "h2_matrix_device_bytes": (C.c_int64, [_P]),
    "h2_free": (None, [_P]),
    "h2_last_error": (C.c_char_p, []),
    "h2_version": (C.c_char_p, []),
}


def load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = load()


class H2Error(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"libh2 status {status}: {msg}")
        self.status = status


def check(status):
    if status != H2_OK:
        raise H2Error(status, lib.h2_last_error().decode(errors="replace"))
