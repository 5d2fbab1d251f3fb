"""TEST INFRASTRUCTURE ONLY — Python wrapper around the CPU oracles.

* ``Oracle("port")`` — our plain-C restatement (oracle/aapdhg_oracle.c,
  built into oracle/build/liboracle.so; compiled on demand with gcc if the
  prebuilt file did not travel).
* ``Oracle("ref")``  — the reference's own sources compiled unmodified into
  oracle/_ref/libaapdhg_ref.so (only where /root/reference was present at
  build time; see oracle/Makefile).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module, and only as the checker.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

from paper_2508_08062_b200 import _abi
from paper_2508_08062_b200.api import (Iterate, KktMetrics, ProblemData, SolveOutput,
                                       SolverConfig, SparseMatrix, StepSizes, check, errbuf,
                                       result_from_c)

ORACLE_DIR = Path(__file__).resolve().parent
PORT_LIB = ORACLE_DIR / "build" / "liboracle.so"
REF_LIB = ORACLE_DIR / "_ref" / "libaapdhg_ref.so"

_dp, _ip = C.POINTER(C.c_double), C.POINTER(C.c_int32)
_E = [C.c_char_p, C.c_size_t]


def build_port(force: bool = False) -> Path:
    if force or not PORT_LIB.exists():
        subprocess.run(["make", "-C", str(ORACLE_DIR), "port"], check=True,
                       stdout=subprocess.DEVNULL)
    return PORT_LIB


def ref_available() -> bool:
    return REF_LIB.exists()


_libs = {}


def _load(kind: str):
    if kind in _libs:
        return _libs[kind]
    if kind == "port":
        lib = C.CDLL(str(build_port()))
        pre = "aapdhg_oracle_"
    elif kind == "ref":
        if not REF_LIB.exists():
            raise FileNotFoundError(f"{REF_LIB} not built (needs /root/reference; make -C oracle ref)")
        lib = C.CDLL(str(REF_LIB))
        pre = "aapdhg_ref_"
    elif kind.startswith("ref-"):  # rounding variants (oracle/Makefile `variants`)
        path = ORACLE_DIR / "_ref" / "variants" / kind[4:] / "libaapdhg_ref.so"
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (make -C oracle variants)")
        lib = C.CDLL(str(path))
        pre = "aapdhg_ref_"
    else:
        raise ValueError(kind)
    PV, SP = C.POINTER(_abi.ProblemView), C.POINTER(_abi.SolveParams)
    f = lambda name, args, res=C.c_int: (setattr(getattr(lib, pre + name), "argtypes", args),
                                        setattr(getattr(lib, pre + name), "restype", res))
    f("solve", [PV, SP, _dp, _dp, C.POINTER(_abi.SolveResultC), _dp, _dp, _dp, _abi.RecordSink,
                C.c_void_p] + _E)
    f("select_step_sizes", [PV, SP, _dp, _dp] + _E)
    f("matvec", [PV, _dp, _dp] + ([] if kind == "port" else _E))
    f("matvec_transpose", [PV, _dp, _dp] + ([] if kind == "port" else _E))
    f("pdhg_step", [PV, C.c_double, C.c_double, _dp, _dp, _dp, _dp] + ([] if kind == "port" else _E))
    f("kkt_metrics", [PV, _dp, _dp, _dp, _dp] + ([] if kind == "port" else _E))
    f("aa_apply", [C.c_int32, C.c_int64, _dp, _dp, C.c_double, _dp, C.c_double, _dp, _dp, _dp]
      + ([] if kind == "port" else _E))
    f("filtered_aa_apply", [C.c_int32, C.c_int64, _dp, _dp, C.c_double, C.c_double, C.c_double,
                            _dp, _dp, _dp, _dp, _ip] + ([] if kind == "port" else _E))
    f("safeguard_pass", [C.c_double, C.c_double, C.c_uint64, C.c_double, C.c_double])
    if kind == "port":
        f("power_norm", [PV, C.c_int32, C.c_double, C.c_uint64, _dp, _ip])
        f("power_start", [C.c_uint64, C.c_int64, _dp], None)
        f("length_bounds", [C.c_int32, _dp, C.c_double, _dp], None)
    else:
        f("power_norm", [PV, C.c_int32, C.c_double, C.c_uint64, _dp] + _E)
        lib.aapdhg_ref_gen.argtypes = [C.c_int32] * 4 + [C.c_uint64, C.c_double, C.c_int32]
        lib.aapdhg_ref_gen.restype = C.c_void_p
        lib.aapdhg_ref_gen_dims.argtypes = [C.c_void_p, _ip, _ip, _ip, C.POINTER(C.c_int64)]
        lib.aapdhg_ref_gen_copy.argtypes = [C.c_void_p, _ip, _ip, _dp, _dp, _dp, _dp, _dp]
        lib.aapdhg_ref_gen_free.argtypes = [C.c_void_p]
    _libs[kind] = (lib, pre)
    return _libs[kind]


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


class Oracle:
    """CPU checker with the same call shapes as paper_2508_08062_b200.Solver."""

    def __init__(self, kind: str = "port"):
        self.kind = kind
        self.lib, self.pre = _load(kind)

    def _fn(self, name):
        return getattr(self.lib, self.pre + name)

    def _e(self):
        return [] if self.kind == "port" else [None, 0]

    def solve(self, p: ProblemData, cfg: SolverConfig, u0: Iterate | None = None) -> SolveOutput:
        n, m = p.n(), p.k.nrows
        view = _abi.problem_view(p)
        prm = cfg.to_params(n + m)
        x, y, lam = np.empty(n), np.empty(m), np.empty(n)
        res = _abi.SolveResultC()
        col = _abi.RecordCollector()
        err = errbuf()
        x0 = _f64(u0.x) if u0 is not None else None
        y0 = _f64(u0.y) if u0 is not None else None
        check(self._fn("solve")(C.byref(view), C.byref(prm), _abi.dptr(x0), _abi.dptr(y0),
                                C.byref(res), _abi.dptr(x), _abi.dptr(y), _abi.dptr(lam), col.cb,
                                None, err, len(err)), err)
        return SolveOutput(result_from_c(res, x, y, lam), col.array())

    def select_step_sizes(self, p: ProblemData, cfg: SolverConfig) -> StepSizes:
        view = _abi.problem_view(p)
        prm = cfg.to_params(p.n() + p.k.nrows)
        tau, sigma = C.c_double(), C.c_double()
        err = errbuf()
        check(self._fn("select_step_sizes")(C.byref(view), C.byref(prm), C.byref(tau),
                                            C.byref(sigma), err, len(err)), err)
        return StepSizes(tau.value, sigma.value)

    def power_norm(self, p: ProblemData, max_iters=5000, rel_tol=1e-4, seed=12345):
        view = _abi.problem_view(p)
        out = C.c_double()
        if self.kind == "port":
            rounds = C.c_int32()
            self._fn("power_norm")(C.byref(view), max_iters, rel_tol, seed, C.byref(out),
                                   C.byref(rounds))
            return out.value, rounds.value
        err = errbuf()
        check(self._fn("power_norm")(C.byref(view), max_iters, rel_tol, seed, C.byref(out), err,
                                     len(err)), err)
        return out.value, None

    def matvec(self, p, x):
        out = np.empty(p.k.nrows)
        self._fn("matvec")(C.byref(_abi.problem_view(p)), _abi.dptr(_f64(x)), _abi.dptr(out),
                           *self._e())
        return out

    def matvec_transpose(self, p, y):
        out = np.empty(p.n())
        self._fn("matvec_transpose")(C.byref(_abi.problem_view(p)), _abi.dptr(_f64(y)),
                                     _abi.dptr(out), *self._e())
        return out

    def pdhg_step(self, p, u: Iterate, s: StepSizes) -> Iterate:
        xn, yn = np.empty(p.n()), np.empty(p.k.nrows)
        self._fn("pdhg_step")(C.byref(_abi.problem_view(p)), s.tau, s.sigma, _abi.dptr(_f64(u.x)),
                              _abi.dptr(_f64(u.y)), _abi.dptr(xn), _abi.dptr(yn), *self._e())
        return Iterate(xn, yn)

    def kkt_metrics(self, p, u: Iterate):
        kkt = np.zeros(4)
        lam = np.empty(p.n())
        self._fn("kkt_metrics")(C.byref(_abi.problem_view(p)), _abi.dptr(_f64(u.x)),
                                _abi.dptr(_f64(u.y)), _abi.dptr(kkt), _abi.dptr(lam), *self._e())
        return KktMetrics(kkt[0], kkt[1], kkt[2]), lam, kkt[3]

    def aa_apply(self, du_cols, dg_cols, u, g, beta=1.0, d_hat=None, eta=1e-10):
        """du_cols/dg_cols: (p, N) arrays, oldest first. Returns (rc, out)."""
        du, dg = _f64(du_cols), _f64(dg_cols)
        p_, N = du.shape
        out = np.empty(N)
        rc = self._fn("aa_apply")(p_, N, _abi.dptr(du), _abi.dptr(dg), beta, _abi.dptr(_f64(d_hat)),
                                  eta, _abi.dptr(_f64(u)), _abi.dptr(_f64(g)), _abi.dptr(out),
                                  *self._e())
        return rc, out

    def filtered_aa_apply(self, e_cols, f_cols, u, g, c_s=0.2, kappa_bar=1e9, beta=1.0,
                          d_hat=None):
        e, f = _f64(e_cols), _f64(f_cols)
        p_, N = e.shape
        out = np.empty(N)
        kept = np.zeros(p_, dtype=np.int32)
        rc = self._fn("filtered_aa_apply")(p_, N, _abi.dptr(e), _abi.dptr(f), c_s, kappa_bar, beta,
                                           _abi.dptr(_f64(d_hat)), _abi.dptr(_f64(u)),
                                           _abi.dptr(_f64(g)), _abi.dptr(out), _abi.iptr(kept),
                                           *self._e())
        return rc, out, kept

    def safeguard_pass(self, g_norm, g0_norm, i, d, eps) -> bool:
        return bool(self._fn("safeguard_pass")(g_norm, g0_norm, i, d, eps))


def power_start(seed: int, n: int) -> np.ndarray:
    lib, _ = _load("port")
    out = np.empty(n)
    lib.aapdhg_oracle_power_start(seed, n, _abi.dptr(out))
    return out


def ref_generate(kind: str, a=0, b=0, c=0, seed=0, slack=0.0, index=0) -> ProblemData:
    """Instances from the reference's own test-support generators
    (proj/tests/support/test_support.cpp:158-283)."""
    lib, _ = _load("ref")
    code = {"toy": 0, "random_box": 1, "transport": 2, "setcover": 3}[kind]
    h = lib.aapdhg_ref_gen(code, a, b, c, seed, slack, index)
    if not h:
        raise RuntimeError("generator failed")
    try:
        n, m1, m2, nnz = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64()
        lib.aapdhg_ref_gen_dims(h, C.byref(n), C.byref(m1), C.byref(m2), C.byref(nnz))
        m = m1.value + m2.value
        rp = np.empty(m + 1, dtype=np.int32)
        ci = np.empty(nnz.value, dtype=np.int32)
        va = np.empty(nnz.value)
        cc, q, l, u = np.empty(n.value), np.empty(m), np.empty(n.value), np.empty(n.value)
        lib.aapdhg_ref_gen_copy(h, _abi.iptr(rp), _abi.iptr(ci), _abi.dptr(va), _abi.dptr(cc),
                                _abi.dptr(q), _abi.dptr(l), _abi.dptr(u))
    finally:
        lib.aapdhg_ref_gen_free(h)
    return ProblemData(SparseMatrix(m, n.value, rp, ci, va), m1.value, cc, q, l, u, name=kind)
