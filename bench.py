"""Benchmark: AA-PDHG fp64 iterations/sec on BASELINE.json configs[4] (the
north-star scaling LP) at every N, with configs[1] as an extra key.

Workload (BASELINE.json configs[4]): planted-optimum LP,
20,000,000 rows x 40,000,000 cols, 10 distinct uniform rows per column (400M
nnz), N(0,1) values, AA-PDHG with memory m = 10, D = 1, eps = 1, beta = 1,
eta = 1e-10, toll = 1e-6 — the largest BASELINE config that fits one B200
and the LP north_star scales over 1/2/4/8 GPUs, so BENCH (N=1) and the
scaling curve share one workload. The `config1` key holds the
same measurements on configs[1] (100k x 200k, 4M nnz, m = 10; "Single GPU")
with its time to 1e-6 KKT. Synthetic seeded data (the reference publishes no
instance files). One "step" = one solver iteration (PDHG map + history push +
safeguard, the AA candidate on accepted steps, KKT records).

Arms
  ours (default)      the sm_100a C-ABI (paper_2508_08062_b200/lib/libaapdhg_cuda.so)
  --impl reference    the reference's own CPU solve() (oracle/_ref, compiled from
                      /root/reference sources; the oracle/ C port if absent)

JSON keys beyond the base contract: roofline (dominant kernel, live CUDA
events), cpu_baseline (the reference on this host's cores), e2e (C-ABI call
from host buffers), time_to_tol (full solve to 1e-6), clocks, gpu_launches.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIG_ID = 4  # the workload (select_workload)
MEMORY = 10
TOLL = 1e-6
GATHER_CEILING = 240.3e9  # measured random-gather rate (profiles/r01/gather.txt)
METRICS = {
    1: "AA-PDHG fp64 iterations/sec (BASELINE configs[1]: 100k x 200k, 4M nnz, m=10)",
    4: "AA-PDHG fp64 iterations/sec (BASELINE configs[4]: 20M x 40M, 400M nnz, m=10)",
}
METRIC = METRICS[4]
WORKLOADS = {
    1: "configs[1] planted LP 100000x200000, 20 nnz/col (4.0M nnz), AA-PDHG m=10, D=1, eps=1, "
       "toll=1e-6",
    4: "configs[4] planted LP 20000000x40000000, 10 nnz/col (400M nnz), AA-PDHG m=10, D=1, "
       "eps=1, toll=1e-6",
}


def select_workload(args, world):
    """configs[4] (the north-star scaling LP) at every N unless --workload
    config1 says otherwise."""
    global CONFIG_ID, METRIC
    CONFIG_ID = 1 if args.workload == "config1" else 4
    METRIC = METRICS[CONFIG_ID]


def load_workload(cfg_id, rank=0, world=1, barrier=None, torch_sort=True):
    """The seeded instance; configs[4] through the on-disk cache
    (problems.cached_config): local rank 0 generates it once, every rank
    memory-maps the same file."""
    from paper_2508_08062_b200 import problems
    if cfg_id != 4:
        return problems.make_config(cfg_id)
    if not torch_sort:  # (the reference arm generates without the GPU)
        os.environ["AAPDHG_GEN_NO_TORCH"] = "1"
    if world > 1 and barrier is not None:
        if int(os.environ.get("LOCAL_RANK", "0")) == 0:
            problems.cached_config(4)
        barrier()
        return problems.cached_config(4, generate=False)
    return problems.cached_config(4)


def host_cpu():
    """'<N>-core <model>' of this host (the CPU baseline's machine)."""
    model = "unknown CPU"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return f"{os.cpu_count()}-core {model}"


def workload_config(p, cfg_id=None):
    cfg_id = CONFIG_ID if cfg_id is None else cfg_id
    return {"workload": WORKLOADS[cfg_id],
            "rows": p.k.nrows, "cols": p.n(), "nnz": p.k.nnz, "memory": MEMORY,
            "l2": "working set > 126 MB L2 (K + K' + history >= 150 MB), no flush"}


def solver_config(tau=0.0, max_iters=100000, reduction="tree", max_wall=3600.0):
    from paper_2508_08062_b200 import Method, SolverConfig
    return SolverConfig(method=Method.AA_PDHG, m=MEMORY, safeguard_d=1.0, safeguard_eps=1.0,
                        toll=TOLL, max_iters=max_iters, tau=tau, sigma=tau, reduction=reduction,
                        max_wall_seconds=max_wall)


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) >= 7:
                    self.samples.append(vals)
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def measured_peak():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(kernel):
    """dram bytes per launch of `kernel` (per iteration for k_plain_loop and
    for configs[4]'s "config4_iteration") from the committed ncu --set full
    captures (profiles/r02d/traffic.json, made by profiles/make_traffic.py;
    the earlier rounds' files for the kernels not re-captured), or None."""
    for rel in ("r02d", "r02b", "r02"):
        try:
            d = json.loads((ROOT / "profiles" / rel / "traffic.json").read_text())[kernel]
        except Exception:
            continue
        if "dram_bytes" in d:
            return float(d["dram_bytes"])
        b = float(d["dram_read_bytes"] + d["dram_write_bytes"])
        return b / d["iterations"] if "iterations" in d else b
    return None


def kernel_bytes(p, name):
    """Algorithmic bytes per launch: CSR streams + compulsory
    gathers (each gathered element counted once) + vector reads/writes."""
    n, m, nnz = p.n(), p.k.nrows, p.k.nnz
    # (the AA history is the ring of g (pipeline.cuh ring_push): one 8-byte
    # store per element and iteration, where the pushed pair read u_{k-1}
    # and stored du, dg)
    if name == "k_dual_side":   # K'y + xhat + KKT dual terms + g_k (x half)
        return 12 * nnz + 4 * (n + 1) + 8 * m + 8 * n * (4 + 1) + 8 * n
    if name == "k_primal_side":  # K xhat + yhat + KKT primal terms + g_k (y half)
        return 12 * nnz + 4 * (m + 1) + 8 * n + 8 * m * (3 + 2) + 8 * m
    if name == "k_plain_loop":  # one plain iteration: both halves
        return kernel_bytes(p, "k_dual_side") + kernel_bytes(p, "k_primal_side")
    if name == "k_spmv_recache":
        return 12 * nnz + 4 * (m + 1) + 8 * n + 8 * m
    if name == "k_spmv_pass":  # mean over the column passes (engine.cu build_blocks)
        per = []
        for rows, cols in ((n, m), (m, n)):  # K' gathers y (m), K gathers x (n)
            nb = -(-cols * 8 // (80 << 20))  # (engine.cu build_blocks: 80 MB blocks
            if cols * 8 <= (64 << 20) or nb < 2:  # above 64 MB vectors)
                continue
            w = -(-cols // nb)
            for b in range(nb - 1):  # the last block is fused into K1 / K2
                per.append(12 * nnz * w / cols + 8 * w + 8 * rows * (1 if b == 0 else 2))
        return sum(per) / len(per) if per else None
    return None


# ---------------------------------------------------------------------------
def cpu_reference_sample(p, tau, iters):
    """The reference CPU solve() on a bounded sample of the workload (explicit
    tau, `iters` iterations). Returns (iterations/s, kind, seconds)."""
    from oracle.pyoracle import Oracle, ref_available
    kind = "reference" if ref_available() else "port"
    orc = Oracle("ref" if kind == "reference" else "port")
    cfg = solver_config(tau=tau, max_iters=iters)
    t0 = time.perf_counter()
    out = orc.solve(p, cfg)
    dt = time.perf_counter() - t0
    return out.result.iterations / dt, kind, dt


def cpu_reference_setup_s(p):
    """The reference's select_step_sizes (seeded power iteration) on this host, seconds."""
    from oracle.pyoracle import Oracle, ref_available
    orc = Oracle("ref" if ref_available() else "port")
    t0 = time.perf_counter()
    orc.select_step_sizes(p, solver_config())
    return time.perf_counter() - t0


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    p = load_workload(CONFIG_ID, torch_sort=False)
    if CONFIG_ID == 4:  # ~50 s per reference iteration: a bounded sample
        args.steps = min(args.steps, 2)
        args.warmup = min(args.warmup, 1)
    from oracle.pyoracle import Oracle, ref_available
    kind = "reference" if ref_available() else "port"
    orc = Oracle("ref" if kind == "reference" else "port")
    # step sizes once (the reference's seeded power iteration), then time
    # `steps` iterations per sample after `warmup` untimed iterations;
    # configs[4]: the reference's own tau from its fixture run
    # (tests/golden/fullsize_cfg4.json, select_step_sizes ~1,000 s on one core)
    tau = None
    if CONFIG_ID == 4:
        try:
            tau = float.fromhex(json.loads(
                (ROOT / "tests" / "golden" / "fullsize_cfg4.json").read_text())["tau"])
        except Exception:
            tau = None
    if tau is None:
        tau = orc.select_step_sizes(p, solver_config()).tau
    iters_per_step = 1
    orc.solve(p, solver_config(tau=tau, max_iters=max(args.warmup, 1)))
    t0 = time.perf_counter()
    out = orc.solve(p, solver_config(tau=tau, max_iters=args.steps * iters_per_step))
    dt = time.perf_counter() - t0
    val = out.result.iterations / dt
    line = {"metric": METRIC, "value": val, "unit": "iterations/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / max(out.result.iterations, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded planted-optimum generator, SURVEY.md 8(d))",
            "config": workload_config(p), "impl": "reference",
            "parallelism": "single (the reference solve is single-threaded)",
            "cpu_baseline": {"value": val, "unit": "iterations/s", "cores": 1, "kind": kind,
                             "host": host_cpu(),
                             "sample": f"{out.result.iterations} iterations of "
                                       f"configs[{CONFIG_ID}] (explicit tau), 1 thread on a "
                                       f"{host_cpu()}: the reference solve() is single-threaded"},
            "e2e": {"value": val, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def pinned_problem(torch, p):
    """A copy of the LP whose arrays live in page-locked host memory, and
    page-locked x / y / lambda result buffers."""
    from paper_2508_08062_b200.api import ProblemData, SparseMatrix

    keep = []

    def pin(a):
        a = np.ascontiguousarray(a)
        t = torch.empty(a.shape, dtype=torch.from_numpy(np.empty(0, a.dtype)).dtype,
                        pin_memory=True)
        keep.append(t)
        v = t.numpy()
        v[...] = a
        return v

    k = SparseMatrix(p.k.nrows, p.k.ncols, pin(p.k.row_ptr), pin(p.k.col_idx), pin(p.k.vals))
    hp = ProblemData(k, p.m1, pin(p.c), pin(p.q), pin(p.l), pin(p.u), name=p.name)
    n, m = p.n(), p.k.nrows
    out = (pin(np.empty(n)), pin(np.empty(m)), pin(np.empty(n)))
    hp._pinned = keep
    return hp, out


def time_e2e(make, cfg, hout, torch, dev, dist=False, tdist=None, reps=3):
    """The e2e leg: a fresh handle from page-locked host buffers (create:
    upload + device ingestion), the solve, the result download; `reps` runs
    (the first one also pays cudaMalloc for block sizes the process has not
    freed yet), the median reported with every run."""
    times, out = [], None
    for _ in range(reps):
        torch.cuda.synchronize(dev)
        if dist:
            tdist.barrier()
        t0 = time.perf_counter()
        s2 = make()
        out = s2.solve(cfg, out=hout)  # x, y, lambda into the pinned buffers, records to host
        dt = time.perf_counter() - t0
        s2.close()  # (freeing device memory is not part of the measured path)
        if dist:
            dt = allreduce_max(tdist, torch, dt, dev)
        times.append(dt)
    return sorted(times)[len(times) // 2], times, out


def allreduce_max(tdist, torch, v, dev):
    """max over ranks (NCCL wants device tensors, gloo host ones)"""
    on = f"cuda:{dev}" if tdist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(v)], dtype=torch.float64, device=on)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    return float(t.item())


def run_ours(args, rank, world, local_rank):
    import ctypes as C

    import torch

    from paper_2508_08062_b200 import Solver, _abi, problems
    from paper_2508_08062_b200.api import check, errbuf

    dev = local_rank
    torch.cuda.set_device(dev)
    dist = world > 1 or args.shard or args.loopback
    if world > 1:
        import torch.distributed as tdist
        p = load_workload(CONFIG_ID, rank, world, barrier=tdist.barrier)
    else:
        p = load_workload(CONFIG_ID)
    if dist:
        import torch.distributed as tdist
        if not tdist.is_initialized():  # --shard at N=1
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            tdist.init_process_group("gloo", rank=0, world_size=1)

    stream = torch.cuda.Stream(device=dev)
    if dist:
        # sharded solve: rank r owns K's row block R_r and
        # column block C_r; exchanges between the phases over peer memory
        # (--transport p2p, the default: the kernels store into every rank's
        # buffers, flag barriers) or NCCL all-gathers (--transport nccl)
        from paper_2508_08062_b200 import DistConfig, nccl_unique_id

        transport = args.transport
        if args.loopback:  # every shard in this process, on this one GPU (a dry run)
            transport = "loopback_p2p" if transport == "p2p" else "loopback"
        elif transport == "p2p":  # every rank must reach every peer (else NCCL)
            ok = world <= 8 and all(torch.cuda.can_device_access_peer(dev, q)
                                    for q in range(torch.cuda.device_count()) if q != dev)
            flag = torch.tensor([1 if ok else 0], dtype=torch.int32,
                                device=f"cuda:{dev}" if tdist.get_backend() == "nccl" else "cpu")
            tdist.all_reduce(flag, op=tdist.ReduceOp.MIN)
            transport = "p2p" if int(flag.item()) else "nccl"
        args.transport = transport

        def dcfg(tr):  # a fresh NCCL id per communicator (ids are single-use)
            if tr.startswith("loopback"):
                return DistConfig(world=args.loopback, rank=0, transport=tr)
            box = [nccl_unique_id() if rank == 0 else None]
            tdist.broadcast_object_list(box, src=0)
            return DistConfig(world=world, rank=rank, transport=tr, nccl_id=box[0])
        t_create = time.perf_counter()
        s = Solver(p, device=dev, dist=dcfg(transport))
        t_create = time.perf_counter() - t_create
        if transport == "p2p" and world > 1:
            # self-check: the peer-memory exchanges must reproduce the NCCL
            # all-gathers bit for bit (same kernels, same data) over 60
            # iterations with AA steps; otherwise run on NCCL
            chk = solver_config(tau=s.select_step_sizes(solver_config()).tau, max_iters=60)
            a = s.solve(chk).trajectory["g_norm"]
            with Solver(p, device=dev, dist=dcfg("nccl")) as s2:
                b = s2.solve(chk).trajectory["g_norm"]
            same = torch.tensor([1 if np.array_equal(a, b) else 0], dtype=torch.int32,
                                device=f"cuda:{dev}" if tdist.get_backend() == "nccl" else "cpu")
            tdist.all_reduce(same, op=tdist.ReduceOp.MIN)
            if not int(same.item()):
                s.close()
                transport = "nccl"
                args.transport = "nccl (p2p self-check failed)"
                s = Solver(p, device=dev, dist=dcfg("nccl"))
    else:
        t_create = time.perf_counter()
        s = Solver(p, device=dev)
        t_create = time.perf_counter() - t_create
    lib = s.lib
    check(lib.aapdhg_cuda_set_stream(s.h, C.c_void_p(stream.cuda_stream)), errbuf())
    tau = s.select_step_sizes(solver_config()).tau

    # warm-up: graph instantiation, caches
    s.solve(solver_config(tau=tau, max_iters=max(args.warmup, 3)))

    # ---- timed: exactly K iterations, inputs resident in HBM ---------------
    # (results land in page-locked host buffers, as in the e2e leg)
    hp, hout = pinned_problem(torch, p)
    cfg = solver_config(tau=tau, max_iters=args.steps)
    if dist:
        tdist.barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        with torch.cuda.stream(stream):
            ev0.record(stream)
            out = s.solve(cfg, out=hout)
            ev1.record(stream)
        torch.cuda.synchronize(dev)
    ms = ev0.elapsed_time(ev1)
    iters = out.result.iterations
    launches, loop_iters = C.c_uint64(), C.c_uint64()
    lib.aapdhg_cuda_last_launch_count(s.h, C.byref(launches), C.byref(loop_iters))
    plain = None
    if not dist:
        pi, ps, pl = C.c_uint64(), C.c_double(), C.c_uint64()
        lib.aapdhg_cuda_last_plain_loop(s.h, C.byref(pi), C.byref(ps), C.byref(pl))
        if pl.value:
            plain = (int(pi.value), float(ps.value), int(pl.value))
    if dist:  # one iteration is one unit of the whole (sharded) job
        ms = allreduce_max(tdist, torch, ms, dev)
    total_iters = float(iters)
    value = total_iters / (ms / 1e3)

    # ---- roofline of the dominant kernel ------------------------------------
    # k_plain_loop from its device clock over the timed region; the per-kernel
    # graph's K1 / K2 (eager launches, CUDA events) beside it
    roofline = None
    if not dist:
        eager = kernel_roofline(args, p, s, lib, tau)
        if plain:
            roofline = plain_loop_roofline(args, p, plain, ms)
            roofline["per_kernel_graph"] = eager
        elif CONFIG_ID == 4:  # the whole iteration (column passes + fused halves)
            roofline = iteration_roofline(p, iters, out.result.i, ms, eager)
        else:
            roofline = eager

    # ---- time to tolerance (full solve to toll 1e-6, step sizes included) --
    ttt = None
    if not args.no_ttt and CONFIG_ID == 1:
        ttt = time_to_tol(args, p, s)
    s.close()

    # ---- e2e: C-ABI call from host buffers (upload + solve + download) -----
    # the LP and the result buffers in page-locked host memory (the base
    # contract's "inputs from pinned host memory"); filled before the clock
    e2e_s, e2e_runs, out2 = time_e2e(
        lambda: (Solver(hp, device=dev, dist=dcfg(transport)) if dist else Solver(hp, device=dev)),
        solver_config(tau=tau, max_iters=args.steps), hout, torch, dev, dist,
        tdist if dist else None)
    h2d = (p.k.row_ptr.nbytes + p.k.col_idx.nbytes + p.k.vals.nbytes + p.c.nbytes + p.q.nbytes
           + p.l.nbytes + p.u.nbytes)
    d2h = (p.n() * 16 + p.k.nrows * 8) + out2.trajectory.nbytes
    e2e = {"value": out2.result.iterations / e2e_s, "unit": "iterations/s",
           "h2d_bytes_per_step": h2d / max(out2.result.iterations, 1),
           "d2h_bytes_per_step": d2h / max(out2.result.iterations, 1),
           "seconds": e2e_s, "runs_s": e2e_runs,
           "path": "aapdhg_cuda_problem_create + aapdhg_cuda_solve (explicit tau) + result "
                   "download; LP and results in page-locked host buffers; median of "
                   f"{len(e2e_runs)} fresh handles"}

    # ---- configs[1] (100k x 200k, 4M nnz) on this one GPU -----------------
    # (before the configs[4] CPU baseline: timed right after that reference run
    # (~30 GB of host memory), the leg's e2e once took 0.1 s instead of 5 ms)
    c1 = None
    if rank == 0 and world == 1 and CONFIG_ID == 4 and not args.no_config1 and not dist:
        c1 = config1_leg(args, torch, dev, stream)

    # ---- CPU baseline on this host (rank 0, N=1 only) ----------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu_iters = 1 if CONFIG_ID == 4 else args.cpu_iters  # (~50 s per configs[4] iteration)
        v, kind, dt = cpu_reference_sample(p, tau, cpu_iters)
        cpu = {"value": v, "unit": "iterations/s", "cores": 1, "kind": kind,
               "host": host_cpu(),
               "sample": f"{cpu_iters} iteration(s) of configs[{CONFIG_ID}] (explicit tau), "
                         f"{dt:.1f} s, 1 thread on a {host_cpu()}: the reference "
                         f"solve() is single-threaded"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "iterations/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / max(iters, 1),
                "higher_is_better": True, "scaling": "strong" if dist else "weak",
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded planted-optimum generator, SURVEY.md 8(d))",
                "config": workload_config(p),
                "parallelism": (f"shard{world} (row/column blocks, "
                                f"{'peer-memory stores + flag barriers' if args.transport == 'p2p' else args.transport})"
                                if dist else "single"),
                "iterations_timed": iters, "aa_steps_timed": out.result.i,
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "time_to_tol": ttt,
                "clocks": clk.summary(), "gpu_launches": int(launches.value),
                "gpu_loop_iterations": int(loop_iters.value),
                "create_s": t_create}
        if args.loopback:
            line["parallelism"] = (f"loopback{args.loopback}: {args.loopback} shards in one "
                                   f"process on one GPU ({args.transport} exchanges) — a dry "
                                   f"run of the sharded path, not a multi-GPU measurement")
        if c1 is not None:
            line["config1"] = c1
        print(json.dumps(line), flush=True)


def iteration_bytes(p, iters, aa_steps, memory=MEMORY):
    """Algorithmic bytes of `iters` iterations of which `aa_steps` took an AA
    step: every iteration K1 + K2 with g_k into the history
    ring; an AA step adds the Gram pass over the window 8N(p+1), the mix
    8N(p+4) (window, u, candidate and its du) and the K x recache
    12 nnz + 4(m+1) + 8n + 8m."""
    n, m, nnz = p.n(), p.k.nrows, p.k.nnz
    N = n + m
    aa = 8 * N * (memory + 1) + 8 * N * (memory + 4) + 12 * nnz + 4 * (m + 1) + 8 * n + 8 * m
    return iters * kernel_bytes(p, "k_plain_loop") + aa_steps * aa


def iteration_roofline(p, iters, aa_steps, ms, eager):
    """configs[4]'s roofline: the algorithmic bytes of the timed iterations
    (iteration_bytes: K1 + K2 with the push per iteration, plus the Gram, the
    mix and the recache per AA step) over the device time of the timed solve
    (CUDA events on the solver's stream); the per-kernel table and the
    dominant kernel's own figure from the eager profile beside it."""
    peak, peak_kind = measured_peak()
    byts = iteration_bytes(p, iters, aa_steps)
    ach = byts / (ms / 1e3) / 1e9
    return {"bound": "hbm", "kernel": "iteration (k_spmv_pass x4 + k_dual_side + k_primal_side"
                                      " per plain step; + AA branch)",
            "achieved": ach, "peak": peak, "peak_source": peak_kind, "unit": "GB/s",
            "frac": ach / peak, "traffic": ncu_traffic("config4_iteration"),
            "traffic_source": "ncu --set full of one plain iteration's kernels, dram bytes "
                              "(profiles/r02d/traffic.json): per plain iteration, against "
                              "bytes_per_plain_iteration",
            "bytes": byts, "bytes_per_plain_iteration": kernel_bytes(p, "k_plain_loop"),
            "timing": "CUDA events on the solver stream around the timed solve",
            "dominant_kernel": eager}


def config1_leg(args, torch, dev, stream):
    """configs[1] (100k x 200k, 4M nnz, AA m=10; BASELINE's "Single GPU"
    config) on this GPU: the same measurements as the headline (resident
    iterations/s, k_plain_loop roofline, e2e from page-locked buffers, the
    reference CPU baseline) plus the time to max KKT <= 1e-6."""
    import ctypes as C

    from paper_2508_08062_b200 import Solver
    from paper_2508_08062_b200.api import check, errbuf
    p = load_workload(1)
    t0 = time.perf_counter()
    s = Solver(p, device=dev)
    create_s = time.perf_counter() - t0
    lib = s.lib
    check(lib.aapdhg_cuda_set_stream(s.h, C.c_void_p(stream.cuda_stream)), errbuf())
    tau = s.select_step_sizes(solver_config()).tau
    # warm-up: graph instantiation and the persistent grid's first partition
    # calibration (engine.cu rebalance: a solve of >= 16 iterations)
    s.solve(solver_config(tau=tau, max_iters=max(args.warmup, 64)))
    steps1 = getattr(args, "steps_cfg1", args.steps)
    hp, hout = pinned_problem(torch, p)
    cfg = solver_config(tau=tau, max_iters=steps1)
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        ev0.record(stream)
        out = s.solve(cfg, out=hout)
        ev1.record(stream)
    torch.cuda.synchronize(dev)
    ms = ev0.elapsed_time(ev1)
    iters = out.result.iterations
    pi, ps, pl = C.c_uint64(), C.c_double(), C.c_uint64()
    lib.aapdhg_cuda_last_plain_loop(s.h, C.byref(pi), C.byref(ps), C.byref(pl))
    eager = kernel_roofline(args, p, s, lib, tau)
    if pl.value:
        roofline = plain_loop_roofline(args, p, (int(pi.value), float(ps.value), int(pl.value)),
                                       ms)
        roofline["per_kernel_graph"] = eager
    else:
        roofline = eager
    # the same roofline in steady state: a 2,000-iteration solve (the 20-step
    # solve above carries the solve's start, one launch per AA step and the
    # dropped speculative K1 of each stop)
    sol = s.solve(solver_config(tau=tau, max_iters=2000))
    lib.aapdhg_cuda_last_plain_loop(s.h, C.byref(pi), C.byref(ps), C.byref(pl))
    if pl.value:
        st = plain_loop_roofline(args, p, (int(pi.value), float(ps.value), int(pl.value)), 1.0)
        roofline["steady_state"] = {
            "iterations": sol.result.iterations, "aa_steps": sol.result.i,
            "plain_iterations": int(pi.value), "launches": int(pl.value),
            "us_per_plain_iteration": 1e6 * float(ps.value) / max(int(pi.value), 1),
            "achieved": st["achieved"], "frac": st["frac"],
            "gather_frac": st["gather_roofline"]["frac"]}
    ttt = None if args.no_ttt else time_to_tol(args, p, s)
    s.close()
    e2e_s, e2e_runs, out2 = time_e2e(lambda: Solver(hp, device=dev),
                                     solver_config(tau=tau, max_iters=steps1), hout, torch, dev)
    h2d = sum(a.nbytes for a in (p.k.row_ptr, p.k.col_idx, p.k.vals, p.c, p.q, p.l, p.u))
    d2h = (p.n() * 16 + p.k.nrows * 8) + out2.trajectory.nbytes
    cpu = None
    if not args.no_cpu:
        v, kind, dt = cpu_reference_sample(p, tau, args.cpu_iters)
        cpu = {"value": v, "unit": "iterations/s", "cores": 1, "kind": kind, "host": host_cpu(),
               "sample": f"{args.cpu_iters} iterations of configs[1] (explicit tau), {dt:.1f} s,"
                         f" 1 thread on a {host_cpu()}: the reference solve() is "
                         f"single-threaded"}
    if cpu is not None and ttt is not None and ttt.get("first_kkt_le_1e-6"):
        # the reference's time to tolerance, extrapolated as
        # its step-size setup + the GPU's iteration count x its s/iteration
        setup = cpu_reference_setup_s(p)
        k_tol = ttt["first_kkt_le_1e-6"]["k"]
        cpu["time_to_tol_extrapolated_s"] = setup + k_tol / cpu["value"]
        cpu["time_to_tol_note"] = (f"extrapolated: select_step_sizes {setup:.1f} s (measured) + "
                                   f"{k_tol} iterations (the GPU's count to max KKT <= 1e-6) "
                                   f"x {1 / cpu['value']:.4f} s per reference iteration")
    return {"metric": METRICS[1], "workload": WORKLOADS[1], "rows": p.k.nrows, "cols": p.n(),
            "nnz": int(p.k.nnz), "value": iters / (ms / 1e3), "unit": "iterations/s",
            "ms_per_step": ms / max(iters, 1), "iterations_timed": iters,
            "aa_steps_timed": out.result.i, "roofline": roofline,
            "e2e": {"value": out2.result.iterations / e2e_s, "unit": "iterations/s",
                    "seconds": e2e_s, "runs_s": e2e_runs,
                    "h2d_bytes_per_step": h2d / max(out2.result.iterations, 1),
                    "d2h_bytes_per_step": d2h / max(out2.result.iterations, 1),
                    "path": "aapdhg_cuda_problem_create + aapdhg_cuda_solve (explicit tau) + "
                            "result download; LP and results in page-locked host buffers; "
                            f"median of {len(e2e_runs)} fresh handles"},
            "cpu_baseline": cpu, "time_to_tol": ttt, "create_s": create_s}


def plain_loop_roofline(args, p, plain, step_ms):
    """Roofline of k_plain_loop, the persistent grid that runs every plain
    iteration of the timed solve, from its own device clock over the timed
    region (globaltimer from each launch's start to its stop, summed by the
    control CTA; aapdhg_cuda_last_plain_loop)."""
    iters, secs, launches = plain
    per_it = kernel_bytes(p, "k_plain_loop")
    achieved = per_it * iters / secs / 1e9
    peak, peak_kind = measured_peak()
    t_it = ncu_traffic("k_plain_loop")
    return {"bound": "hbm", "kernel": "k_plain_loop", "achieved": achieved, "peak": peak,
            "peak_source": peak_kind, "unit": "GB/s", "frac": achieved / peak,
            "traffic": (t_it * iters / launches) if (t_it and args.traffic is None)
            else args.traffic,
            "traffic_source": "ncu --set full of one k_plain_loop launch (profiles/r02d/"
                              "traffic.json), dram bytes per iteration x iterations per launch",
            "bytes_per_launch": per_it * iters / launches,
            "bytes_per_iteration": per_it,
            "avg_launch_us": 1e6 * secs / launches,
            "iterations_per_launch": iters / launches,
            "launches": launches,
            "timing": "device globaltimer inside the timed region (launch start -> stop)",
            "share_of_step": secs / (step_ms / 1e3),
            "gather_roofline": {
                "bound": "random 8-byte gathers (L1TEX sectors)",
                "ceiling_gather_per_s": GATHER_CEILING,
                "ceiling_source": "profiles/r01/gather.txt: 4M random gathers from an "
                                  "L2-resident vector, 16.6 us on this pool's B200",
                "gathers_per_iteration": 2 * int(p.k.nnz),
                "achieved_gather_per_s": 2 * p.k.nnz * iters / secs,
                "frac": 2 * p.k.nnz * iters / secs / GATHER_CEILING}}


def kernel_roofline(args, p, s, lib, tau):
    import ctypes as C
    lib.aapdhg_cuda_set_profiling(s.h, 1)
    s.solve(solver_config(tau=tau, max_iters=min(args.steps, 400)))
    names = C.create_string_buffer(4096)
    msa = (C.c_double * 64)()
    la = (C.c_uint64 * 64)()
    cnt = C.c_int32()
    lib.aapdhg_cuda_kernel_times(s.h, names, 4096, msa, la, 64, C.byref(cnt))
    lib.aapdhg_cuda_set_profiling(s.h, 0)
    kn = names.value.decode().split("\n")[: cnt.value]
    kstats = {kn[i]: (msa[i], la[i]) for i in range(cnt.value)}
    tot_ms = sum(v[0] for v in kstats.values())
    dom = max((k for k in kstats if kernel_bytes(p, k)), key=lambda k: kstats[k][0])
    avg_ms = kstats[dom][0] / kstats[dom][1]
    peak, peak_kind = measured_peak()
    achieved = kernel_bytes(p, dom) / (avg_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                "peak_source": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                "traffic": args.traffic if args.traffic is not None else ncu_traffic(dom),
                "traffic_source": "ncu --set full (profiles/r02/traffic.json), cold caches",
                "bytes_per_launch": kernel_bytes(p, dom),
                "avg_launch_us": avg_ms * 1e3,
                "share_of_step": kstats[dom][0] / tot_ms if tot_ms else None,
                "per_kernel_us": {k: 1e3 * v[0] / max(v[1], 1) for k, v in kstats.items()}}

    # the bound that actually binds: random 8-byte gathers of
    # x[col], one per nonzero, against the measured B200 ceiling
    gr = {}
    for k in ("k_dual_side", "k_primal_side"):
        if k in kstats and "k_spmv_pass" not in kstats:  # (blocked: a launch gathers one block)
            us = 1e3 * kstats[k][0] / max(kstats[k][1], 1)
            gr[k] = {"gathers_per_launch": int(p.k.nnz), "avg_launch_us": us,
                     "achieved_gather_per_s": p.k.nnz / (us * 1e-6),
                     "frac": p.k.nnz / (us * 1e-6) / GATHER_CEILING}
    roofline["gather_roofline"] = {
        "bound": "random 8-byte gathers (L1TEX sectors)", "ceiling_gather_per_s": GATHER_CEILING,
        "ceiling_source": "profiles/r01/gather.txt: 4M random gathers from an L2-resident "
                          "vector, 16.6 us on this pool's B200 (1.21 cycles/gather/SM)",
        "kernels": gr}
    return roofline


def time_to_tol(args, p, s):
    t0 = time.perf_counter()
    full = s.solve(solver_config(max_wall=args.ttt_cap))
    ttt = {"seconds": time.perf_counter() - t0, "iterations": full.result.iterations,
           "aa_steps": full.result.i, "status": full.result.status.name,
           "objective": full.result.objective,
           "planted_objective": getattr(p, "planted_objective", None),
           "max_kkt": full.result.kkt.max()}
    kk = full.trajectory
    if kk.size:
        mk = np.maximum(np.maximum(kk["r_gap"], kk["r_primal"]), kk["r_dual"])
        hit = np.flatnonzero(mk <= 1e-6)
        if hit.size:
            ttt["first_kkt_le_1e-6"] = {"k": int(kk["k"][hit[0]]),
                                        "elapsed_s": float(kk["elapsed_s"][hit[0]])}
    return ttt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed iterations (default: 200 for configs[4], 20,000 for configs[1])")
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-iters", type=int, default=20)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ttt", action="store_true")
    ap.add_argument("--ttt-cap", type=float, default=60.0)
    ap.add_argument("--transport", choices=["p2p", "nccl"], default="p2p",
                    help="sharded-solve exchanges: peer-memory stores (p2p, <= 8 GPUs) or NCCL")
    ap.add_argument("--shard", action="store_true",
                    help="use the sharded solve even at N=1 (exercises the N>1 path)")
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu dram bytes per launch of the dominant kernel, if captured")
    ap.add_argument("--workload", choices=["config4", "config1"], default="config4",
                    help="the timed LP (configs[4] at every N by default)")
    ap.add_argument("--loopback", type=int, default=0,
                    help="dry run of the sharded solve: K in-process shards on this one GPU")
    ap.add_argument("--no-config1", action="store_true",
                    help="skip the configs[1] leg of the N=1 line")
    args = ap.parse_args()
    if args.impl == "reference":
        # bounded CPU sample: <= 500 iterations (~20 s of reference work at
        # ~40 ms per iteration); the driver's --steps 20 --warmup 5 run as given
        args.warmup = max(args.warmup, 0)
        args.steps = min(args.steps if args.steps is not None else 500, 500)
        args.warmup = min(args.warmup, 50)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    select_workload(args, world)
    # no --steps: a run that ends within minutes — configs[4] 200 iterations
    # (~1.5 s timed, the e2e leg as many), the configs[1] leg its 20,000
    args.steps_cfg1 = args.steps if args.steps is not None else 20000
    if args.steps is None:
        args.steps = 200 if CONFIG_ID == 4 else 20000
    if world > 1 and args.impl == "ours":
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(local_rank)
        tdist.init_process_group("nccl")
    try:
        if args.impl == "reference":
            run_reference_arm(args, rank, world)
        else:
            run_ours(args, rank, world, local_rank)
    finally:
        if world > 1 and args.impl == "ours":
            import torch.distributed as tdist
            tdist.destroy_process_group()


if __name__ == "__main__":
    main()
