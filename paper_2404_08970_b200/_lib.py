"""ctypes view of include/gwdp.h (argument marshalling only).

Loads the in-tree ``libgwdp.so`` and fails loudly if it is missing: there is no CPU
fallback anywhere in the product path.
"""

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libgwdp.so")

GW_OK = 0
STATUS = {
    0: "GW_OK", 1: "GW_ERR_INVALID_ARG", 2: "GW_ERR_DIM_MISMATCH", 3: "GW_ERR_UNSORTED",
    4: "GW_ERR_NEGATIVE_WEIGHT", 5: "GW_ERR_NOT_NORMALIZED", 6: "GW_ERR_NONFINITE", 7: "GW_ERR_CONFIG",
    8: "GW_ERR_UNSUPPORTED", 9: "GW_ERR_OOM", 10: "GW_ERR_CUDA", 11: "GW_ERR_NCCL",
}
GW_LOSS_SQUARE = 0
GW_F32, GW_F64 = 0, 1
GW_NO_VALIDATE = 0x1
GW_HOST_VECTORS = 0x2
GW_GRID2D = 0x4
GW_SOLVE_TRACE_OBJECTIVE = 0x1

# exported symbols (include/gwdp.h) -- checked by tests/test_abi.py
SYMBOLS = [
    "gw_ctx_create", "gw_ctx_destroy", "gw_ctx_trim", "gw_ctx_profile", "gw_last_error", "gw_abi_version",
    "gw_get_unique_id", "gw_comm_init", "gw_comm_init_host", "gw_comm_destroy", "gw_shard_rows", "gw_check_shards",
    "gw_grad_dp", "sinkhorn_solve", "entropic_gw_solve", "fgw_solve", "ugw_solve", "gw_solve_set_export",
]


class GwError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        self.code = STATUS.get(status, str(status))
        super().__init__("%s: %s" % (self.code, msg))


class gw_problem(C.Structure):
    _fields_ = [("n", C.c_int64), ("m", C.c_int64), ("row0", C.c_int64), ("n_local", C.c_int64),
                ("x", C.c_void_p), ("y", C.c_void_p), ("p", C.c_void_p), ("q", C.c_void_p),
                ("k", C.c_int32), ("loss", C.c_int32), ("dtype", C.c_int32), ("flags", C.c_uint32)]


class gw_moments(C.Structure):
    _fields_ = [("row_sum", C.c_void_p), ("row_ysum", C.c_void_p),
                ("col_sum", C.c_void_p), ("col_xsum", C.c_void_p)]


class gw_sinkhorn_opts(C.Structure):
    _fields_ = [("eps", C.c_double), ("max_iter", C.c_int32), ("tol", C.c_double), ("check_every", C.c_int32)]


class gw_sinkhorn_info(C.Structure):
    _fields_ = [("iters", C.c_int32), ("converged", C.c_int32), ("fused_iters", C.c_int32),
                ("marginal_violation", C.c_double)]


class gw_solve_opts(C.Structure):
    _fields_ = [("eps", C.c_double), ("tau", C.c_double), ("outer_iters", C.c_int32),
                ("inner", gw_sinkhorn_opts), ("flags", C.c_uint32)]


class gw_result(C.Structure):
    _fields_ = [("gw_objective", C.c_double), ("entropic_objective", C.c_double),
                ("marginal_violation", C.c_double), ("outer_iters", C.c_int32),
                ("inner_iters_total", C.c_int32), ("converged", C.c_int32), ("inner_fused_total", C.c_int32),
                ("ms_grad", C.c_double), ("ms_sinkhorn", C.c_double), ("ms_total", C.c_double),
                ("grad_onepass_total", C.c_int32)]


# int (*gw_allgather_fn)(const void *send, void *recv, int64_t bytes, void *user)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)

_lib = None


def load(path=LIB_PATH):
    """Load libgwdp.so (raises if it is missing -- build it with __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError("libgwdp.so not found at %s: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)" % path)
    lib = C.CDLL(path)
    P = C.c_void_p
    i64 = C.c_int64
    lib.gw_ctx_create.argtypes = [C.POINTER(P), C.c_int, P, P]
    lib.gw_ctx_destroy.argtypes = [P]
    lib.gw_ctx_trim.argtypes = [P]
    lib.gw_ctx_profile.argtypes = [P, C.c_int, P, P, C.c_int]
    lib.gw_last_error.restype = C.c_char_p
    lib.gw_abi_version.restype = C.c_int
    lib.gw_get_unique_id.argtypes = [C.c_char_p]
    lib.gw_comm_init.argtypes = [C.POINTER(P), C.c_char_p, C.c_int, C.c_int]
    lib.gw_comm_destroy.argtypes = [P]
    lib.gw_comm_init_host.argtypes = [C.POINTER(P), C.c_int, C.c_int, ALLGATHER_FN, P]
    lib.gw_shard_rows.argtypes = [i64, C.c_int, C.c_int, C.POINTER(i64), C.POINTER(i64)]
    lib.gw_check_shards.argtypes = [C.POINTER(i64), C.c_int, i64]
    lib.gw_grad_dp.argtypes = [P, C.POINTER(gw_problem), P, i64, P, i64, C.POINTER(gw_moments)]
    lib.sinkhorn_solve.argtypes = [P, C.POINTER(gw_problem), P, i64, C.POINTER(gw_sinkhorn_opts), P, P, P, i64,
                                   C.POINTER(gw_sinkhorn_info)]
    lib.entropic_gw_solve.argtypes = [P, C.POINTER(gw_problem), C.POINTER(gw_solve_opts), P, P, i64, P, P,
                                      C.POINTER(gw_result), P]
    lib.fgw_solve.argtypes = [P, C.POINTER(gw_problem), P, P, C.c_double, C.POINTER(gw_solve_opts), P, P, i64, P, P,
                              C.POINTER(gw_result), P]
    lib.ugw_solve.argtypes = [P, C.POINTER(gw_problem), C.c_double, C.POINTER(gw_solve_opts), P, P, i64, P, P,
                              C.POINTER(gw_result), P]
    lib.gw_solve_set_export.argtypes = [P, C.c_int32, P, P, i64]
    for name in SYMBOLS:
        f = getattr(lib, name)
        if f.restype is None or f.restype is C.c_int:
            if name not in ("gw_last_error", "gw_abi_version"):
                f.restype = C.c_int
    _lib = lib
    return lib


def check(status):
    if status != GW_OK:
        raise GwError(status, load().gw_last_error().decode(errors="replace"))
