"""ctypes mirror of the C-ABI in ``include/aapdhg_cuda.h``.

Only POD layouts and the loader live here. The product library is
``paper_2508_08062_b200/lib/libaapdhg_cuda.so`` (built by
``__graft_entry__.build()``); loading fails loudly when it is missing — there
is no CPU fallback on the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
LIB_DIR = PKG_DIR / "lib"
CUDA_LIB = LIB_DIR / "libaapdhg_cuda.so"
HOST_LIB = LIB_DIR / "libaapdhg.so"

ABI_VERSION = 3

# aapdhg_status
OK, ERR_INPUT, ERR_DIMENSION, ERR_UNSUPPORTED, ERR_SINGULAR, ERR_CUDA, ERR_INTERNAL = range(7)
# methods / statuses / reduction modes
METHOD_PDHG, METHOD_AA, METHOD_FAA = 0, 1, 2
(SOLVE_RESIDUAL_TOL, SOLVE_KKT_TOL, SOLVE_MAX_ITERS, SOLVE_TIMEOUT,
 SOLVE_FIXED_POINT_START) = range(5)
REDUCE_AUTO, REDUCE_SERIAL, REDUCE_TREE = 0, 1, 2
# sharded-solve transports
DIST_NCCL, DIST_LOOPBACK, DIST_P2P, DIST_LOOPBACK_P2P = 0, 1, 2, 3
NCCL_ID_BYTES = 128

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


class CsrView(C.Structure):
    _fields_ = [("nrows", C.c_int32), ("ncols", C.c_int32), ("nnz", C.c_int64),
                ("row_ptr", _ip), ("col_idx", _ip), ("vals", _dp)]


class ProblemView(C.Structure):
    _fields_ = [("k", CsrView), ("m1", C.c_int32), ("c", _dp), ("q", _dp),
                ("l", _dp), ("u", _dp)]


class DistView(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("transport", C.c_int32),
                ("pad0", C.c_int32), ("nccl_id", C.POINTER(C.c_uint8))]


class SolveParams(C.Structure):
    _fields_ = [("method", C.c_int32), ("reduction", C.c_int32), ("m", C.c_uint64),
                ("safeguard_d", C.c_double), ("safeguard_eps", C.c_double),
                ("beta", C.c_double), ("d_hat", _dp), ("eta", C.c_double),
                ("c_s", C.c_double), ("kappa_bar", C.c_double), ("toll", C.c_double),
                ("kkt_eps", C.c_double), ("kkt_terminate", C.c_int32), ("pad0", C.c_int32),
                ("max_iters", C.c_uint64), ("max_wall_seconds", C.c_double),
                ("tau", C.c_double), ("sigma", C.c_double)]


class Record(C.Structure):
    _fields_ = [("k", C.c_uint64), ("g_norm", C.c_double), ("aa_step", C.c_int32),
                ("pad0", C.c_int32), ("i", C.c_uint64), ("j", C.c_uint64),
                ("r_gap", C.c_double), ("r_primal", C.c_double), ("r_dual", C.c_double),
                ("objective", C.c_double), ("elapsed_s", C.c_double)]


RECORD_DTYPE = np.dtype([("k", "<u8"), ("g_norm", "<f8"), ("aa_step", "<i4"), ("pad0", "<i4"),
                         ("i", "<u8"), ("j", "<u8"), ("r_gap", "<f8"), ("r_primal", "<f8"),
                         ("r_dual", "<f8"), ("objective", "<f8"), ("elapsed_s", "<f8")])
assert RECORD_DTYPE.itemsize == C.sizeof(Record)


class SolveResultC(C.Structure):
    _fields_ = [("status", C.c_int32), ("pad0", C.c_int32), ("iterations", C.c_uint64),
                ("i", C.c_uint64), ("j", C.c_uint64), ("aa_failures", C.c_uint64),
                ("g_norm", C.c_double), ("r_gap", C.c_double), ("r_primal", C.c_double),
                ("r_dual", C.c_double), ("objective", C.c_double), ("tau", C.c_double),
                ("sigma", C.c_double), ("wall_seconds", C.c_double)]


RecordSink = C.CFUNCTYPE(None, C.POINTER(Record), C.c_uint64, C.c_void_p)


def dptr(a):
    """double* of a contiguous float64 array (None -> NULL)."""
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def iptr(a):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_ip)


class RecordCollector:
    """Accumulates streamed records into one numpy structured array."""

    def __init__(self):
        self.chunks = []
        self.cb = RecordSink(self._sink)

    def _sink(self, recs, count, _ctx):
        if count:
            buf = C.string_at(recs, int(count) * RECORD_DTYPE.itemsize)
            self.chunks.append(np.frombuffer(buf, dtype=RECORD_DTYPE).copy())

    def array(self):
        if not self.chunks:
            return np.zeros(0, dtype=RECORD_DTYPE)
        return np.concatenate(self.chunks)


def csr_view(k):
    """CsrView over a SparseMatrix-like object (arrays kept alive by k)."""
    return CsrView(int(k.nrows), int(k.ncols), int(k.nnz), iptr(k.row_ptr), iptr(k.col_idx),
                   dptr(k.vals))


def problem_view(prob):
    """ProblemView over a ProblemData-like object (arrays kept alive by prob)."""
    k = prob.k
    v = ProblemView()
    v.k = CsrView(int(k.nrows), int(k.ncols), int(k.nnz), iptr(k.row_ptr), iptr(k.col_idx),
                  dptr(k.vals))
    v.m1 = int(prob.m1)
    v.c, v.q, v.l, v.u = dptr(prob.c), dptr(prob.q), dptr(prob.l), dptr(prob.u)
    return v


def _declare_cuda(lib):
    H = C.c_void_p
    E = [C.c_char_p, C.c_size_t]
    sig = {
        "aapdhg_cuda_abi_version": ([], C.c_int),
        "aapdhg_cuda_device_info": ([C.c_char_p, C.c_size_t], C.c_int),
        "aapdhg_cuda_problem_create": ([C.POINTER(ProblemView), C.c_int, C.POINTER(H)] + E, C.c_int),
        "aapdhg_cuda_problem_destroy": ([H], C.c_int),
        "aapdhg_cuda_problem_dims": ([H, _ip, _ip, _ip, C.POINTER(C.c_int64)], C.c_int),
        "aapdhg_cuda_solve": ([H, C.POINTER(SolveParams), _dp, _dp, C.POINTER(SolveResultC),
                               _dp, _dp, _dp, RecordSink, C.c_void_p] + E, C.c_int),
        "aapdhg_cuda_select_step_sizes": ([H, C.POINTER(SolveParams), _dp, _dp] + E, C.c_int),
        "aapdhg_cuda_power_norm": ([H, C.c_int32, C.c_double, C.c_uint64, C.c_int32, _dp, _ip]
                                   + E, C.c_int),
        "aapdhg_cuda_matvec": ([H, _dp, _dp] + E, C.c_int),
        "aapdhg_cuda_matvec_transpose": ([H, _dp, _dp] + E, C.c_int),
        "aapdhg_cuda_pdhg_step": ([H, C.c_double, C.c_double, _dp, _dp, _dp, _dp] + E, C.c_int),
        "aapdhg_cuda_kkt_metrics": ([H, C.c_int32, _dp, _dp, _dp, _dp] + E, C.c_int),
        "aapdhg_cuda_aa_apply": ([H, C.c_int32, C.c_int32, _dp, _dp, C.c_double, _dp,
                                  C.c_double, _dp, _dp, _dp] + E, C.c_int),
        "aapdhg_cuda_filtered_aa_apply": ([H, C.c_int32, C.c_int32, _dp, _dp, C.c_double,
                                           C.c_double, C.c_double, _dp, _dp, _dp, _dp, _ip]
                                          + E, C.c_int),
        "aapdhg_cuda_workspace_create": ([C.c_int32, C.c_int64, C.POINTER(H)] + E, C.c_int),
        "aapdhg_cuda_faa_op": ([H, C.c_int32, C.c_int32, _dp, _dp, C.c_double, C.c_double,
                                C.c_double, _dp, C.c_int32, _dp, _dp, _dp, _ip] + E, C.c_int),
        "aapdhg_cuda_economy_qr": ([H, C.c_int32, C.c_int32, _dp, _dp, _dp] + E, C.c_int),
        "aapdhg_cuda_csr_from_triplets": ([C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                           C.c_int64, C.c_void_p, _ip, C.c_void_p, _ip, _ip,
                                           _dp, C.POINTER(C.c_int64)] + E, C.c_int),
        "aapdhg_cuda_set_stream": ([H, C.c_void_p], C.c_int),
        "aapdhg_cuda_set_profiling": ([H, C.c_int32], C.c_int),
        "aapdhg_cuda_kernel_times": ([H, C.c_char_p, C.c_size_t, _dp,
                                      C.POINTER(C.c_uint64), C.c_int32, _ip], C.c_int),
        "aapdhg_cuda_nccl_id": ([C.POINTER(C.c_uint8), C.c_size_t] + E, C.c_int),
        "aapdhg_cuda_partition": ([C.POINTER(CsrView), C.c_int32, _ip, _ip], C.c_int),
        "aapdhg_cuda_balance_partition": ([C.c_int32, C.c_int32, _ip, _dp, _ip, _ip, _ip],
                                          C.c_int),
        "aapdhg_cuda_problem_create_dist": ([C.POINTER(ProblemView), C.c_int, C.POINTER(DistView),
                                             C.POINTER(H)] + E, C.c_int),
        "aapdhg_cuda_last_launch_count": ([H, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)],
                                          C.c_int),
        "aapdhg_cuda_last_plain_loop": ([H, C.POINTER(C.c_uint64), _dp, C.POINTER(C.c_uint64)],
                                        C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


# every symbol include/aapdhg_cuda.h declares
CUDA_SYMBOLS = (
    "aapdhg_cuda_abi_version", "aapdhg_cuda_device_info", "aapdhg_cuda_problem_create",
    "aapdhg_cuda_problem_destroy", "aapdhg_cuda_problem_dims", "aapdhg_cuda_solve",
    "aapdhg_cuda_select_step_sizes", "aapdhg_cuda_power_norm", "aapdhg_cuda_matvec",
    "aapdhg_cuda_matvec_transpose", "aapdhg_cuda_pdhg_step", "aapdhg_cuda_kkt_metrics",
    "aapdhg_cuda_aa_apply", "aapdhg_cuda_filtered_aa_apply", "aapdhg_cuda_workspace_create",
    "aapdhg_cuda_faa_op", "aapdhg_cuda_economy_qr", "aapdhg_cuda_csr_from_triplets",
    "aapdhg_cuda_set_stream",
    "aapdhg_cuda_set_profiling",
    "aapdhg_cuda_kernel_times", "aapdhg_cuda_last_launch_count", "aapdhg_cuda_last_plain_loop",
    "aapdhg_cuda_nccl_id", "aapdhg_cuda_partition", "aapdhg_cuda_problem_create_dist",
    "aapdhg_cuda_balance_partition",
)

_cuda_lib = None


def cuda_lib():
    """Load the sm_100a library. Raises (no fallback) when it is absent."""
    global _cuda_lib
    if _cuda_lib is None:
        path = Path(os.environ.get("AAPDHG_CUDA_LIB", CUDA_LIB))
        if not path.exists():
            raise RuntimeError(
                f"CUDA extension {path} is missing: run __graft_entry__.build() "
                "(there is no CPU fallback on the product path)")
        lib = C.CDLL(str(path), mode=C.RTLD_GLOBAL)
        _declare_cuda(lib)
        if lib.aapdhg_cuda_abi_version() != ABI_VERSION:
            raise RuntimeError("libaapdhg_cuda.so ABI version mismatch")
        _cuda_lib = lib
    return _cuda_lib
