"""Host-side mirror of the reference solver API, over the sm_100a C-ABI.

Names, defaults, argument meaning and error behaviour follow the reference
C++ interface:

* ``Method`` / ``SolveStatus``      — proj/include/aapdhg/solver.hpp:15-23
* ``SolverConfig``                  — proj/include/aapdhg/solver.hpp:25-39
* ``AAParams`` / ``FilterParams``   — proj/include/aapdhg/anderson.hpp:21-25,
                                      proj/include/aapdhg/filtering.hpp:14-17
* ``KktMetrics``, ``TrajectoryRecord``, ``SolveResult``, ``SolveOutput``
                                    — proj/include/aapdhg/solver.hpp:41-78
* ``solve(p, cfg[, u0])``           — proj/include/aapdhg/solver.hpp:93-99
* ``select_step_sizes``, ``kkt_metrics``, ``safeguard_pass``
                                    — proj/include/aapdhg/solver.hpp:81-91
* exceptions                        — proj/include/aapdhg/errors.hpp:8-30

Every compute call goes through ``libaapdhg_cuda.so``; nothing here computes
the path on the CPU.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Optional

import numpy as np

from . import _abi


# ---- errors (errors.hpp:8-30) ----------------------------------------------
class Error(RuntimeError):
    pass


class InputError(Error):
    pass


class UnsupportedError(Error):
    pass


class SingularError(Error):
    pass


class DimensionError(Error):
    pass


class CudaError(Error):
    pass


_ERR = {_abi.ERR_INPUT: InputError, _abi.ERR_DIMENSION: DimensionError,
        _abi.ERR_UNSUPPORTED: UnsupportedError, _abi.ERR_SINGULAR: SingularError,
        _abi.ERR_CUDA: CudaError, _abi.ERR_INTERNAL: Error}


def check(rc: int, err: C.Array) -> None:
    if rc != _abi.OK:
        raise _ERR.get(rc, Error)(err.value.decode(errors="replace") or f"error code {rc}")


def errbuf():
    return C.create_string_buffer(512)


# ---- model types ------------------------------------------------------------
class Method(IntEnum):
    PDHG = _abi.METHOD_PDHG
    AA_PDHG = _abi.METHOD_AA
    FAA_PDHG = _abi.METHOD_FAA


class SolveStatus(IntEnum):
    RESIDUAL_TOL = _abi.SOLVE_RESIDUAL_TOL
    KKT_TOL = _abi.SOLVE_KKT_TOL
    MAX_ITERS = _abi.SOLVE_MAX_ITERS
    TIMEOUT = _abi.SOLVE_TIMEOUT
    FIXED_POINT_START = _abi.SOLVE_FIXED_POINT_START


REDUCTIONS = {"auto": _abi.REDUCE_AUTO, "serial": _abi.REDUCE_SERIAL, "tree": _abi.REDUCE_TREE}


@dataclass
class SparseMatrix:
    """CSR, int32 row_ptr/col_idx + fp64 vals (sparse_linalg.hpp:18-28)."""
    nrows: int
    ncols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    vals: np.ndarray

    def __post_init__(self):
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.int32)
        self.col_idx = np.ascontiguousarray(self.col_idx, dtype=np.int32)
        self.vals = np.ascontiguousarray(self.vals, dtype=np.float64)
        if self.row_ptr.shape != (self.nrows + 1,):
            raise DimensionError("SparseMatrix: row_ptr size")

    @property
    def nnz(self) -> int:
        return int(self.vals.shape[0])

    @staticmethod
    def from_triplets(nrows, ncols, rows, cols, vals) -> "SparseMatrix":
        """Sort by (row, col) and sum duplicates (sparse_linalg.cpp:11-42)."""
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        vals = np.asarray(vals, dtype=np.float64)
        if rows.size and (rows.min() < 0 or rows.max() >= nrows or cols.min() < 0
                          or cols.max() >= ncols):
            raise DimensionError("from_triplets: entry out of range")
        order = np.lexsort((cols, rows))  # stable: duplicates keep input order
        rows, cols, vals = rows[order], cols[order], vals[order]
        if rows.size:
            key = rows * ncols + cols
            first = np.ones(rows.size, dtype=bool)
            first[1:] = key[1:] != key[:-1]
            if not first.all():
                # sequential left-to-right duplicate sum, as the reference
                starts = np.flatnonzero(first)
                out = np.empty(starts.size)
                for t, s in enumerate(starts):
                    e = starts[t + 1] if t + 1 < starts.size else rows.size
                    acc = 0.0
                    for v in vals[s:e]:
                        acc += v
                    out[t] = acc
                rows, cols, vals = rows[starts], cols[starts], out
        row_ptr = np.zeros(nrows + 1, dtype=np.int64)
        np.add.at(row_ptr, rows + 1, 1)
        return SparseMatrix(nrows, ncols, np.cumsum(row_ptr), cols, vals)

    def transpose(self) -> "SparseMatrix":
        """CSR of the transpose; entries of each row in ascending original row."""
        rows = np.repeat(np.arange(self.nrows, dtype=np.int32), np.diff(self.row_ptr))
        order = np.argsort(self.col_idx, kind="stable")
        cnt = np.bincount(self.col_idx, minlength=self.ncols)
        rp = np.zeros(self.ncols + 1, dtype=np.int64)
        rp[1:] = np.cumsum(cnt)
        return SparseMatrix(self.ncols, self.nrows, rp, rows[order], self.vals[order])

    def dense(self) -> np.ndarray:
        out = np.zeros((self.nrows, self.ncols))
        rows = np.repeat(np.arange(self.nrows), np.diff(self.row_ptr))
        np.add.at(out, (rows, self.col_idx), self.vals)
        return out


def vstack(a: SparseMatrix, b: SparseMatrix) -> SparseMatrix:
    """Stacks b below a (sparse_linalg.cpp:44-58)."""
    if a.ncols != b.ncols:
        raise DimensionError("vstack: column count mismatch")
    rp = np.concatenate([a.row_ptr, a.row_ptr[-1] + b.row_ptr[1:]])
    return SparseMatrix(a.nrows + b.nrows, a.ncols, rp, np.concatenate([a.col_idx, b.col_idx]),
                        np.concatenate([a.vals, b.vals]))


@dataclass
class ProblemData:
    """min c'x s.t. Gx >= h, Ax = b, l <= x <= u via K = [G; A], q = [h; b]
    (lp_model.hpp:32-53). ``m1`` = rows of G."""
    k: SparseMatrix
    m1: int
    c: np.ndarray
    q: np.ndarray
    l: np.ndarray
    u: np.ndarray
    name: str = ""
    maximize: bool = False

    def __post_init__(self):
        for f in ("c", "q", "l", "u"):
            setattr(self, f, np.ascontiguousarray(getattr(self, f), dtype=np.float64))
        if self.c.shape != (self.k.ncols,) or self.l.shape != self.c.shape \
                or self.u.shape != self.c.shape or self.q.shape != (self.k.nrows,):
            raise DimensionError("ProblemData: vector sizes do not match K")
        if not 0 <= self.m1 <= self.k.nrows:
            raise DimensionError("ProblemData: bad m1")

    def n(self) -> int:
        return self.k.ncols

    def m2(self) -> int:
        return self.k.nrows - self.m1

    @property
    def h(self):
        return self.q[: self.m1]

    @property
    def b(self):
        return self.q[self.m1:]


@dataclass
class Iterate:
    x: np.ndarray
    y: np.ndarray


@dataclass
class StepSizes:
    tau: float = 0.0
    sigma: float = 0.0


@dataclass
class AAParams:
    beta: float = 1.0
    d_hat: Optional[np.ndarray] = None  # None = identity
    eta: float = 1e-10


@dataclass
class FilterParams:
    c_s: float = 0.2
    kappa_bar: float = 1e9


@dataclass
class SolverConfig:
    method: Method = Method.PDHG
    m: int = 5
    safeguard_d: float = 1.0
    safeguard_eps: float = 1.0
    aa: AAParams = field(default_factory=AAParams)
    filter: FilterParams = field(default_factory=FilterParams)
    toll: float = 1e-4
    kkt_eps: float = 1e-4
    kkt_terminate: bool = False
    max_iters: int = 100000
    max_wall_seconds: float = 3600.0
    tau: float = 0.0
    sigma: float = 0.0
    # B200 extension: reduction order ("auto" | "serial" | "tree"), see
    # include/aapdhg_cuda.h. "serial" reproduces the CPU reference bitwise.
    reduction: str = "auto"

    def to_params(self, N: int) -> _abi.SolveParams:
        if self.reduction not in REDUCTIONS:
            raise InputError(f"reduction must be one of {sorted(REDUCTIONS)}")
        p = _abi.SolveParams()
        p.method = int(self.method)
        p.reduction = REDUCTIONS[self.reduction]
        p.m = int(self.m) if self.m >= 0 else 0
        p.safeguard_d = self.safeguard_d
        p.safeguard_eps = self.safeguard_eps
        p.beta = self.aa.beta
        self._d_hat = None
        if self.aa.d_hat is not None and len(self.aa.d_hat):
            self._d_hat = np.ascontiguousarray(self.aa.d_hat, dtype=np.float64)
            if self._d_hat.shape != (N,):
                raise DimensionError("aa: d_hat size mismatch")
            p.d_hat = _abi.dptr(self._d_hat)
        p.eta = self.aa.eta
        p.c_s = self.filter.c_s
        p.kappa_bar = self.filter.kappa_bar
        p.toll = self.toll
        p.kkt_eps = self.kkt_eps
        p.kkt_terminate = 1 if self.kkt_terminate else 0
        p.max_iters = int(self.max_iters)
        p.max_wall_seconds = self.max_wall_seconds
        p.tau = self.tau
        p.sigma = self.sigma
        return p


@dataclass
class KktMetrics:
    r_gap: float = 0.0
    r_primal: float = 0.0
    r_dual: float = 0.0

    def max(self) -> float:
        return max(self.r_gap, self.r_primal, self.r_dual)


@dataclass
class SolveResult:
    status: SolveStatus
    u: Iterate
    lambda_: np.ndarray
    iterations: int
    i: int
    j: int
    aa_failures: int
    g_norm: float
    kkt: KktMetrics
    objective: float
    steps: StepSizes
    wall_seconds: float


@dataclass
class SolveOutput:
    result: SolveResult
    trajectory: np.ndarray  # structured array, fields of TrajectoryRecord


def result_from_c(res: _abi.SolveResultC, x, y, lam) -> SolveResult:
    return SolveResult(
        status=SolveStatus(res.status), u=Iterate(x, y), lambda_=lam,
        iterations=int(res.iterations), i=int(res.i), j=int(res.j),
        aa_failures=int(res.aa_failures), g_norm=res.g_norm,
        kkt=KktMetrics(res.r_gap, res.r_primal, res.r_dual), objective=res.objective,
        steps=StepSizes(res.tau, res.sigma), wall_seconds=res.wall_seconds)


def safeguard_pass(g_norm: float, g0_norm: float, i: int, d: float, eps: float) -> bool:
    """||g|| <= D ||g0|| (i+1)^-(1+eps), equality passes (solver.cpp:59-62).
    Scalar host predicate; the solve loop evaluates it on the device from a
    host-built (i+1)^-(1+eps) table so both agree bitwise."""
    return g_norm <= d * g0_norm * math.pow(float(i) + 1.0, -(1.0 + eps))


@dataclass
class DistConfig:
    """A sharded solve (include/aapdhg_cuda.h aapdhg_dist_view): `world`
    row/column blocks of the LP. transport "nccl": this process is shard
    `rank` on its own GPU, all ranks pass the same `nccl_id` (nccl_unique_id()
    on rank 0, broadcast by the caller). "p2p": as "nccl", but inside the
    iteration the kernels store straight into every shard's buffers over peer
    memory (CUDA IPC, NVLink) and each exchange is a flag barrier (<= 8
    shards). "loopback" / "loopback_p2p": all shards in this process on one
    device with copy / peer-store exchanges (the partitioned path on one GPU)."""
    world: int
    rank: int = 0
    transport: str = "nccl"
    nccl_id: Optional[bytes] = None


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (rank 0 of a sharded solve)."""
    lib = _abi.cuda_lib()
    buf = (C.c_uint8 * _abi.NCCL_ID_BYTES)()
    err = errbuf()
    check(lib.aapdhg_cuda_nccl_id(buf, len(buf), err, len(err)), err)
    return bytes(buf)


def partition(k: SparseMatrix, world: int):
    """Row / column block bounds of a `world`-way sharded solve (host only)."""
    lib = _abi.cuda_lib()
    view = _abi.csr_view(k)
    rows = np.zeros(world + 1, dtype=np.int32)
    cols = np.zeros(world + 1, dtype=np.int32)
    rc = lib.aapdhg_cuda_partition(C.byref(view), int(world), _abi.iptr(rows), _abi.iptr(cols))
    if rc == _abi.ERR_UNSUPPORTED:
        raise UnsupportedError("partition: every shard needs at least one row and one column")
    if rc:
        raise InputError("partition: bad arguments")
    return rows, cols


class Solver:
    """A problem resident in HBM (one device handle); reusable across solves
    (the reference's sweep mode re-solves one ProblemData many times).
    With `dist`, this process's part of a sharded multi-GPU solve: solve()
    and select_step_sizes() are then collective over the ranks."""

    def __init__(self, p: ProblemData, device: int = 0, dist: Optional[DistConfig] = None):
        self.p = p
        self.lib = _abi.cuda_lib()
        self._view = _abi.problem_view(p)
        h = C.c_void_p()
        err = errbuf()
        if dist is None:
            check(self.lib.aapdhg_cuda_problem_create(C.byref(self._view), int(device),
                                                       C.byref(h), err, len(err)), err)
        else:
            dv = _abi.DistView()
            dv.rank = int(dist.rank)
            dv.world = int(dist.world)
            transports = {"nccl": _abi.DIST_NCCL, "loopback": _abi.DIST_LOOPBACK,
                          "p2p": _abi.DIST_P2P, "loopback_p2p": _abi.DIST_LOOPBACK_P2P}
            if dist.transport not in transports:
                raise InputError("dist: transport must be one of " + ", ".join(transports))
            dv.transport = transports[dist.transport]
            self._id = None
            if dist.nccl_id is not None:
                self._id = (C.c_uint8 * _abi.NCCL_ID_BYTES).from_buffer_copy(
                    bytes(dist.nccl_id).ljust(_abi.NCCL_ID_BYTES, b"\0"))
                dv.nccl_id = C.cast(self._id, C.POINTER(C.c_uint8))
            check(self.lib.aapdhg_cuda_problem_create_dist(C.byref(self._view), int(device),
                                                            C.byref(dv), C.byref(h), err,
                                                            len(err)), err)
        self.h = h

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.aapdhg_cuda_problem_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def N(self) -> int:
        return self.p.n() + self.p.k.nrows

    def solve(self, cfg: SolverConfig, u0: Optional[Iterate] = None,
              out: Optional[tuple] = None) -> SolveOutput:
        """``out`` = (x[n], y[m], lambda[n]) float64 buffers to fill (e.g.
        page-locked host memory: the results are then DMA'd straight into
        them); fresh arrays otherwise."""
        n, m = self.p.n(), self.p.k.nrows
        prm = cfg.to_params(n + m)
        if out is not None:
            x, y, lam = out
            for a, sz in ((x, n), (y, m), (lam, n)):
                if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.shape == (sz,)
                        and a.flags.c_contiguous and a.flags.writeable):
                    raise DimensionError("solve: out buffers must be writable float64 (n, m, n)")
        else:
            x = np.empty(n)
            y = np.empty(m)
            lam = np.empty(n)
        x0 = y0 = None
        if u0 is not None:
            x0 = np.ascontiguousarray(u0.x, dtype=np.float64)
            y0 = np.ascontiguousarray(u0.y, dtype=np.float64)
            if x0.shape != (n,) or y0.shape != (m,):
                raise DimensionError("solve: start iterate dims mismatch")
        res = _abi.SolveResultC()
        col = _abi.RecordCollector()
        err = errbuf()
        check(self.lib.aapdhg_cuda_solve(self.h, C.byref(prm), _abi.dptr(x0), _abi.dptr(y0),
                                         C.byref(res), _abi.dptr(x), _abi.dptr(y), _abi.dptr(lam),
                                         col.cb, None, err, len(err)), err)
        return SolveOutput(result_from_c(res, x, y, lam), col.array())

    def select_step_sizes(self, cfg: SolverConfig) -> StepSizes:
        prm = cfg.to_params(self.N)
        tau, sigma = C.c_double(), C.c_double()
        err = errbuf()
        check(self.lib.aapdhg_cuda_select_step_sizes(self.h, C.byref(prm), C.byref(tau),
                                                     C.byref(sigma), err, len(err)), err)
        return StepSizes(tau.value, sigma.value)

    def kkt_metrics(self, u: Iterate, reduction: str = "auto"):
        kkt = np.zeros(4)
        lam = np.empty(self.p.n())
        err = errbuf()
        check(self.lib.aapdhg_cuda_kkt_metrics(
            self.h, REDUCTIONS[reduction], _abi.dptr(np.ascontiguousarray(u.x, dtype=np.float64)),
            _abi.dptr(np.ascontiguousarray(u.y, dtype=np.float64)), _abi.dptr(kkt),
            _abi.dptr(lam), err, len(err)), err)
        return KktMetrics(kkt[0], kkt[1], kkt[2]), lam

    def pdhg_step(self, u: Iterate, s: StepSizes) -> Iterate:
        xn = np.empty(self.p.n())
        yn = np.empty(self.p.k.nrows)
        err = errbuf()
        check(self.lib.aapdhg_cuda_pdhg_step(
            self.h, s.tau, s.sigma, _abi.dptr(np.ascontiguousarray(u.x, dtype=np.float64)),
            _abi.dptr(np.ascontiguousarray(u.y, dtype=np.float64)), _abi.dptr(xn),
            _abi.dptr(yn), err, len(err)), err)
        return Iterate(xn, yn)


@dataclass
class SweepCase:
    cfg: SolverConfig
    name: str


def sweep_cases(base: SolverConfig, d=(), eps=(), m=(), kappa_bar=()) -> list:
    """The CLI's --sweep-D/--sweep-eps/--sweep-m/--sweep-kappa-bar cross
    product with its case names (proj/src/cli.cpp:155-180)."""
    import copy
    out = []
    for vd in (d or [None]):
        for ve in (eps or [None]):
            for vm in (m or [None]):
                for vk in (kappa_bar or [None]):
                    c = copy.deepcopy(base)
                    parts = []
                    if vd is not None:
                        c.safeguard_d = vd
                        parts.append("D%g" % vd)
                    if ve is not None:
                        c.safeguard_eps = ve
                        parts.append("eps%g" % ve)
                    if vm is not None:
                        c.m = int(vm)
                        parts.append("m%d" % int(vm))
                    if vk is not None:
                        c.filter = FilterParams(c_s=c.filter.c_s, kappa_bar=vk)
                        parts.append("kappa%g" % vk)
                    out.append(SweepCase(c, "_".join(parts)))
    return out


def solve_sweep(p: ProblemData, cases, workers: int = 0, devices=(0,)) -> list:
    """Sweep mode (proj/src/cli.cpp:184-209): the cases on `workers` threads
    (AAPDHG_SWEEP_WORKERS when 0), each keeping one resident handle on its
    device (round-robin) and taking cases from a shared counter; several
    workers per GPU run concurrently on their own streams. Returns
    (ok, error, SolveOutput | None) per case, in case order."""
    import itertools
    import os
    import threading
    cases = list(cases)
    if not devices:
        raise InputError("solve_sweep: no devices")
    if workers <= 0:
        workers = max(1, int(os.environ.get("AAPDHG_SWEEP_WORKERS", "1") or 1))
    workers = max(1, min(workers, len(cases)))
    out = [None] * len(cases)
    counter = itertools.count()
    lock = threading.Lock()

    def work(w):
        try:
            s = Solver(p, devices[w % len(devices)])
        except Error as e:
            s, err = None, str(e)
        try:
            while True:
                with lock:
                    idx = next(counter)
                if idx >= len(cases):
                    return
                if s is None:
                    out[idx] = (False, err, None)
                    continue
                c = cases[idx].cfg if isinstance(cases[idx], SweepCase) else cases[idx]
                try:
                    out[idx] = (True, "", s.solve(c))
                except Error as e:
                    out[idx] = (False, str(e), None)
        finally:
            if s is not None:
                s.close()

    threads = [threading.Thread(target=work, args=(w,)) for w in range(workers)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    return out


def solve(p: ProblemData, cfg: SolverConfig, u0: Optional[Iterate] = None,
          device: int = 0) -> SolveOutput:
    """solve(p, cfg[, u0]) — proj/include/aapdhg/solver.hpp:93-99."""
    with Solver(p, device) as s:
        return s.solve(cfg, u0)


def select_step_sizes(p: ProblemData, cfg: SolverConfig, device: int = 0) -> StepSizes:
    """select_step_sizes — proj/include/aapdhg/solver.hpp:89-91."""
    with Solver(p, device) as s:
        return s.select_step_sizes(cfg)


def kkt_metrics(u: Iterate, p: ProblemData, device: int = 0):
    """kkt_metrics — proj/include/aapdhg/solver.hpp:85-87; returns (KktMetrics, lambda)."""
    with Solver(p, device) as s:
        return s.kkt_metrics(u)
