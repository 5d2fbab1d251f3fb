"""Seeded synthetic LP instances standing in for BASELINE.json's configs.

The reference publishes no benchmark files for this path; the
MIPLIB instances of the paper are not available. These generators follow
SURVEY.md §8(d) (shapes, sparsity, value distributions, planted optimum).
Each config is generated from ``numpy.random.Generator(PCG64(2508080620+cfg))``
so the oracle and the GPU path always see bit-identical inputs.

Problem form for the planted configs: G empty (m1 = 0), A = the matrix,
l = 0, u = +inf (Lambda tags all NONNEG).
"""
from __future__ import annotations

import numpy as np

from .api import ProblemData, SparseMatrix

SEED_BASE = 2508080620

CONFIGS = {
    0: dict(kind="planted", m=1_000, n=2_000, nnz=20_000, method="aa", memory=5),
    1: dict(kind="planted", m=100_000, n=200_000, per_col=20, method="aa", memory=10),
    2: dict(kind="transport", sources=2_000, sinks=2_000, method="faa", memory=10,
            c_s=float(np.sqrt(1.0 - 0.99 ** 2)), kappa_bar=1e4),
    3: dict(kind="zipf", m=2_000_000, n=4_000_000, alpha=1.5, cap=10_000, method="aa",
            memory=20),
    4: dict(kind="planted", m=20_000_000, n=40_000_000, per_col=10, method="aa", memory=10),
}


def _argsort_stable(key: np.ndarray, use_torch: bool | None = None) -> np.ndarray:
    """The stable sorting permutation of int64 keys — unique whatever sort
    produces it (equal keys keep their input order) — on a CUDA device when
    one is present and the array is large (config 3/4: 150-400M keys,
    minutes in numpy), numpy otherwise. use_torch forces the torch path
    (tests compare the two)."""
    import os
    if use_torch is None:
        use_torch = key.size > (16 << 20) and os.environ.get("AAPDHG_GEN_NO_TORCH") != "1"
    if use_torch:
        try:
            import torch
            dev = "cuda" if torch.cuda.is_available() else None
            if dev is not None or use_torch is True:
                t = torch.from_numpy(key)
                if dev is not None and key.size > (16 << 20):
                    t = t.cuda()
                order = torch.argsort(t, stable=True)
                del t
                out = order.cpu().numpy()
                del order
                if dev is not None:
                    torch.cuda.empty_cache()
                return out
        except Exception:  # no usable torch / device: the numpy sort below
            pass
    return np.argsort(key, kind="stable")


_argsort_distinct = _argsort_stable


def _csr_from_coo(m, n, rows, cols, vals) -> SparseMatrix:
    """CSR with columns ascending in each row (entries distinct)."""
    key = rows.astype(np.int64) * np.int64(n) + cols.astype(np.int64)
    if key.size > 1 and not bool(np.all(key[1:] > key[:-1])):
        order = _argsort_distinct(key)  # = lexsort((cols, rows)): keys distinct
        del key
        rows, cols, vals = rows[order], cols[order], vals[order]
        del order
    else:
        del key
    rp = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=m), out=rp[1:])
    return SparseMatrix(m, n, rp.astype(np.int32), cols.astype(np.int32), vals)


def _distinct_per_group(rng, groups: int, k, universe: int):
    """For each group g draw k[g] distinct uniform values in [0, universe)."""
    k = np.broadcast_to(np.asarray(k, dtype=np.int64), (groups,))
    total = int(k.sum())
    grp = np.repeat(np.arange(groups, dtype=np.int64), k)
    val = rng.integers(0, universe, size=total, dtype=np.int64)
    if total and int(k.min()) == int(k.max()):
        # equal group sizes: the same draws and redraws as the general loop
        # below, sorting each group in place (groups are already contiguous)
        w = int(k[0])
        v = val.reshape(groups, w)
        while True:
            v.sort(axis=1)
            dup = np.zeros_like(v, dtype=bool)
            dup[:, 1:] = v[:, 1:] == v[:, :-1]
            nd = int(dup.sum())
            if nd == 0:
                return grp, v.reshape(-1)
            v[dup] = rng.integers(0, universe, size=nd, dtype=np.int64)
    while True:
        # = np.lexsort((val, grp)): one stable sort of the combined key
        order = _argsort_stable(grp * np.int64(universe) + val)
        g2, v2 = grp[order], val[order]
        dup = np.zeros(total, dtype=bool)
        dup[1:] = (g2[1:] == g2[:-1]) & (v2[1:] == v2[:-1])
        nd = int(dup.sum())
        grp, val = g2, v2
        if nd == 0:
            return grp, val
        val[dup] = rng.integers(0, universe, size=nd, dtype=np.int64)


def _plant(rng, k: SparseMatrix, name: str) -> ProblemData:
    """Planted optimum: x*_j = 0 on a Bernoulli(1/2) half, else U(0,1);
    y* ~ N(0,1); s*_j ~ U(0,1) where x*_j = 0; b = A x*, c = A'y* + s*."""
    m, n = k.nrows, k.ncols
    zero = rng.random(n) < 0.5
    xs = np.where(zero, 0.0, rng.random(n))
    ys = rng.standard_normal(m)
    ss = np.where(zero, rng.random(n), 0.0)
    rows = np.repeat(np.arange(m), np.diff(k.row_ptr))
    b = np.bincount(rows, weights=k.vals * xs[k.col_idx], minlength=m)
    c = np.bincount(k.col_idx, weights=k.vals * ys[rows], minlength=n) + ss
    p = ProblemData(k, 0, c, b, np.zeros(n), np.full(n, np.inf), name=name)
    p.planted_objective = float(c @ xs)
    p.planted_x, p.planted_y = xs, ys
    return p


def planted(m: int, n: int, seed: int, nnz: int | None = None, per_col: int | None = None,
            name: str = "planted") -> ProblemData:
    rng = np.random.default_rng(seed)
    if nnz is not None:
        pos = rng.choice(m * n, size=nnz, replace=False)
        rows, cols = pos // n, pos % n
    else:
        cols, rows = _distinct_per_group(rng, n, per_col, m)
    vals = rng.standard_normal(rows.size)
    return _plant(rng, _csr_from_coo(m, n, rows, cols, vals), name)


def transport(sources: int, sinks: int, seed: int) -> ProblemData:
    """Rows 0..S-1: supply sum_j x_ij = s_i; rows S..S+T-1: demand
    sum_i x_ij = d_j; column i*T + j has two 1.0 entries; s, d ~ U(1,100),
    d rescaled to sum(s) with the rounding absorbed in the last d; c ~ U(0,1)."""
    rng = np.random.default_rng(seed)
    S, T = sources, sinks
    n = S * T
    s = rng.uniform(1.0, 100.0, S)
    d = rng.uniform(1.0, 100.0, T)
    d = d * (s.sum() / d.sum())
    d[-1] = s.sum() - d[:-1].sum()
    c = rng.random(n)
    col = np.arange(n, dtype=np.int64)
    rows = np.concatenate([col // T, S + col % T])
    cols = np.concatenate([col, col])
    k = _csr_from_coo(S + T, n, rows, cols, np.ones(2 * n))
    return ProblemData(k, 0, c, np.concatenate([s, d]), np.zeros(n), np.full(n, np.inf),
                       name="transport")


def zipf_planted(m: int, n: int, alpha: float, cap: int, seed: int) -> ProblemData:
    rng = np.random.default_rng(seed)
    support = np.arange(1, cap + 1, dtype=np.float64)
    pmf = support ** (-alpha)
    cdf = np.cumsum(pmf / pmf.sum())
    lengths = np.minimum(np.searchsorted(cdf, rng.random(m), side="right") + 1, cap)
    rows, cols = _distinct_per_group(rng, m, lengths, n)
    vals = rng.standard_normal(rows.size)
    return _plant(rng, _csr_from_coo(m, n, rows, cols, vals), "zipf")


def make_config(cfg: int, scale: float = 1.0) -> ProblemData:
    """Instance for BASELINE.json configs[cfg]; ``scale`` < 1 shrinks the
    row/column counts (same density per row/column) for quick tests."""
    spec = CONFIGS[cfg]
    seed = SEED_BASE + cfg
    if spec["kind"] == "planted":
        m, n = max(2, int(spec["m"] * scale)), max(4, int(spec["n"] * scale))
        if "nnz" in spec:
            return planted(m, n, seed, nnz=max(1, int(spec["nnz"] * scale * scale)),
                           name=f"config{cfg}")
        return planted(m, n, seed, per_col=min(spec["per_col"], m), name=f"config{cfg}")
    if spec["kind"] == "transport":
        S = max(2, int(spec["sources"] * scale))
        T = max(2, int(spec["sinks"] * scale))
        return transport(S, T, seed)
    if spec["kind"] == "zipf":
        m, n = max(2, int(spec["m"] * scale)), max(4, int(spec["n"] * scale))
        return zipf_planted(m, n, spec["alpha"], min(spec["cap"], n), seed)
    raise ValueError(cfg)


def toy() -> ProblemData:
    """min 0*x s.t. x = 3, x >= 0 (proj/data/toy.mps)."""
    k = SparseMatrix(1, 1, np.array([0, 1]), np.array([0]), np.array([1.0]))
    return ProblemData(k, 0, np.zeros(1), np.array([3.0]), np.zeros(1), np.full(1, np.inf),
                       name="toy")


# ---------------------------------------------------------------------------
# On-disk instances (config 4 takes minutes to generate and ~5 GB): generated
# once per box into a cache directory and memory-mapped by every process
# that needs it (every rank of a sharded run maps the same pages).

GENERATOR_VERSION = 1  # bump when a generator's output changes


def cache_dir(cfg: int, scale: float = 1.0) -> "Path":
    import os
    from pathlib import Path
    root = Path(os.environ.get("AAPDHG_INSTANCE_CACHE", "/tmp/aapdhg_instances"))
    return root / f"cfg{cfg}_s{scale:g}_v{GENERATOR_VERSION}"


_FIELDS = ("row_ptr", "col_idx", "vals", "c", "q", "l", "u")


def save_instance(p: ProblemData, d) -> None:
    """Writes the arrays as .npy files, then a `complete` marker (written
    last, so a reader never maps a half-written instance)."""
    import json
    d.mkdir(parents=True, exist_ok=True)
    arrays = dict(row_ptr=p.k.row_ptr, col_idx=p.k.col_idx, vals=p.k.vals, c=p.c, q=p.q,
                  l=p.l, u=p.u)
    for k, a in arrays.items():
        np.save(d / f"{k}.npy.tmp.npy", a)
        (d / f"{k}.npy.tmp.npy").replace(d / f"{k}.npy")
    meta = dict(m=int(p.k.nrows), n=int(p.k.ncols), m1=int(p.m1), name=p.name,
                planted_objective=getattr(p, "planted_objective", None))
    (d / "meta.json").write_text(json.dumps(meta))
    (d / "complete").write_text("ok")


def load_instance(d) -> ProblemData:
    """Memory-maps a saved instance (read-only pages, shared between processes)."""
    import json
    meta = json.loads((d / "meta.json").read_text())
    a = {k: np.load(d / f"{k}.npy", mmap_mode="r") for k in _FIELDS}
    k = SparseMatrix(meta["m"], meta["n"], a["row_ptr"], a["col_idx"], a["vals"])
    p = ProblemData(k, meta["m1"], a["c"], a["q"], a["l"], a["u"], name=meta["name"])
    if meta.get("planted_objective") is not None:
        p.planted_objective = meta["planted_objective"]
    return p


def cached_config(cfg: int, scale: float = 1.0, generate: bool = True) -> ProblemData:
    """make_config(cfg, scale) through the on-disk cache: generated (by the
    caller with generate=True) when absent, memory-mapped afterwards."""
    d = cache_dir(cfg, scale)
    if not (d / "complete").exists():
        if not generate:
            raise FileNotFoundError(f"instance {d} is not generated yet")
        save_instance(make_config(cfg, scale), d)
    return load_instance(d)
