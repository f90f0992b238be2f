"""Benchmark driver (contract: DESIGN.md §Measurement).

Headline workload = BASELINE.json's metric as quoted on config 3:
TI-Sinkhorn (H variant) on two seeded 8-component 2-D Gaussian mixtures,
N = M = 65536, fp32 log-domain, eps = 1e-2 * max|x - y|^2, KL rho = 1.
A "step" is one solve of that configuration through the public API -- 200
H-Sinkhorn iterations (g half-step + f half-step each) over the whole problem
from zero potentials, as BASELINE config 3 states it; ``value`` = iterations/s
of the whole job = 200 * steps / timed seconds (an L2 flush between steps is
inside the timed region).  With
``--gpus N`` under torchrun the single problem is row-sharded across the
ranks (one NCCL all-gather per iteration) and the step time is the max over
ranks.  The same line carries the other BASELINE configs as ``secondary``
entries (batched FW cfg2, barycenter cfg5, cfg1, cfg4), each sharded by
problem across ranks with no communication.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--no-secondary]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TI-Sinkhorn iter/s (N=M=65536, d=2)"
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2
CFG3_ITERS = 200  # BASELINE config 3: one solve = 200 iterations
CFG2_BYTES_PER_ITER = 268435456  # 4096 * 32 * (1024 + 1024)
CFG5_BYTES_PER_ITER = 268435456  # 64 * 16 * 8192 * 32


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured (MEASURED_PEAKS.json)"
    except OSError:
        return ({"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": None},
                "fallback (B200_PROFILING.md)")


PROBES_PATH = os.path.join(ROOT, "profiles", "r2_probes.json")


def load_probes():
    """Committed MUFU / DFMA probe results (scripts/run_probes.py on a B200):
    the FIXED denominators of the exp-bound rooflines."""
    try:
        with open(PROBES_PATH) as fh:
            pr = json.load(fh)
        return {"ex2_per_s": pr["ex2"]["per_s_median"], "dfma_per_s": pr["dfma"]["per_s_median"],
                "source": "profiles/r2_probes.json (uot_probe_mufu_ex2 / uot_probe_dfma, "
                          f"median at {pr['ex2']['clocks'].get('sm_mhz')} MHz)"}
    except (OSError, KeyError, ValueError):
        # nominal: 16 ex2/clk/SM and 64 DFMA/clk/SM x 148 SMs x 1965 MHz
        return {"ex2_per_s": 16 * 148 * 1.965e9, "dfma_per_s": 64 * 148 * 1.965e9,
                "source": "nominal (no committed probe file)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}

        def num(v):
            try:
                return float(v)
            except ValueError:
                return None

        sm = [v for v in (num(r[1]) for r in self.rows) if v is not None]
        mx = [v for v in (num(r[2]) for r in self.rows) if v is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[5 + k] == "Active"})
        busy = [v for v in sm if v > 0.5 * max(sm)] if sm else []
        pw = [v for v in (num(r[3]) for r in self.rows) if v is not None]
        return {"sm_mhz": float(np.median(busy or sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows), "power_w": float(np.median(pw)) if pw else None}


def cuda_timer():
    import torch

    st = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)

    class T:
        def __enter__(self):
            e0.record(st)
            return self

        def __exit__(self, *exc):
            e1.record(st)
            torch.cuda.synchronize()
            self.ms = e0.elapsed_time(e1)

    return T()


def max_over_ranks(v, world, dev):
    if world == 1:
        return v
    import torch

    t = torch.tensor([float(v)], device=dev)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# CPU baselines: the oracle port (fp64 restatement of the reference path,
# oracle/) timed on the box's host cores on a bounded sample.


def host_cores():
    return len(os.sched_getaffinity(0))


CFG3_SAMPLE_COLS = 4096


def cpu_cfg3(c, cols=CFG3_SAMPLE_COLS):
    import oracle as O

    threads = host_cores()
    os.environ["ORACLE_THREADS"] = str(threads)
    rng = np.random.default_rng(1)
    sel = np.sort(rng.choice(len(c.y), cols, replace=False))
    cost = O.PointCost(c.x, c.y[sel])
    t0 = time.perf_counter()
    cost.smin_cols(np.zeros(len(c.x)), c.eps, c.alpha)
    el = time.perf_counter() - t0
    pairs = len(c.x) * cols
    rate = 1.0 / (el / pairs * 2.0 * len(c.x) * len(c.y))
    sample = (f"one g half-step restricted to {cols} of {len(c.y)} columns x {len(c.x)} rows "
              f"({pairs:.3g} pair evaluations, fp64 C oracle restating sinkhorn.py:93-100 over "
              f"entropies.py:84-92, {threads} threads), extrapolated to 2*N*M pairs/iteration")
    cpu_cfg3.last_seconds = el
    return rate, threads, sample


def _fw_worker(args):
    os.environ["OMP_NUM_THREADS"] = "1"
    import oracle as O
    from paper_2201_00730_b200 import synthetic as S

    idx, iters = args
    x, y, a, b = S.cfg2_batch(batch=4096, start=idx, count=1)
    t0 = time.perf_counter()
    O.fw_fixed(x[0], y[0], a[0], b[0], 1.0, 1.0, iters)
    return time.perf_counter() - t0


def cpu_cfg2(iters=20):
    """cores problems x `iters` line-search FW iterations (oracle port of
    fw.py:176-232 with the reference's ternary search), one process per core;
    throughput scaled to the full 4096-problem batched iteration."""
    import multiprocessing as mp

    cores = host_cores()
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(cores) as pool:
        pool.map(_fw_worker, [(k, iters) for k in range(cores)])
    wall = time.perf_counter() - t0
    problem_iters_per_s = cores * iters / wall
    rate = problem_iters_per_s / 4096.0
    sample = (f"{cores} cfg2 problems x {iters} line-search FW iterations (numpy/C oracle port, "
              f"one process per core), scaled to 4096 problems per batched iteration")
    return rate, cores, sample


def _bary_worker(args):
    os.environ["OMP_NUM_THREADS"] = "1"
    import oracle as O
    from paper_2201_00730_b200 import synthetic as S

    idx, iters = args
    xs, ws = S.cfg5_batch(start=idx, count=1)
    t0 = time.perf_counter()
    O.fw_barycenter_fixed(list(xs[0]), list(ws[0]), np.full(16, 1 / 16), 1.0, iters)
    return time.perf_counter() - t0


def cpu_cfg5(iters=2):
    import multiprocessing as mp

    cores = min(host_cores(), 64)
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(cores) as pool:
        pool.map(_bary_worker, [(k, iters) for k in range(cores)])
    wall = time.perf_counter() - t0
    rate = cores * iters / wall / 64.0
    sample = (f"{cores} cfg5 problems x {iters} FW iterations (oracle port of "
              f"barycenter.py:361-411), scaled to 64 problems per batched iteration")
    return rate, cores, sample


def cpu_cfg4(cols=1024):
    """cfg4: one g half-step of problem 0 restricted to `cols` columns (fp64
    oracle, d = 64 squared Euclidean computed directly), all host threads;
    scaled to 2 x 256 x 4096 x 4096 pair evaluations per batched iteration."""
    import oracle as O
    from paper_2201_00730_b200 import synthetic as S

    threads = host_cores()
    os.environ["ORACLE_THREADS"] = str(threads)
    x, y, a, b = S.cfg4_batch(count=1)
    cost = O.PointCost(x[0], y[0][:cols])
    t0 = time.perf_counter()
    cost.smin_cols(np.zeros(x.shape[1]), S.CFG4_EPS, a[0])
    el = time.perf_counter() - t0
    pairs = x.shape[1] * cols
    rate = 1.0 / (el / pairs * 2.0 * 256 * x.shape[1] * y.shape[1])
    sample = (f"one g half-step of problem 0 restricted to {cols} of {y.shape[1]} columns "
              f"({pairs:.3g} pairs, d=64, fp64 C oracle, {threads} threads), extrapolated to "
              f"2*B*N*M pairs per batched iteration")
    return rate, threads, sample


def cpu_cfg1(iters=1000):
    """cfg1: the oracle port's H-Sinkhorn on one core, `iters` iterations."""
    import oracle as O
    from paper_2201_00730_b200 import synthetic as S

    os.environ["ORACLE_THREADS"] = "1"
    c = S.cfg1_inputs()
    cost = O.PointCost(c.x, c.y, p=2.0, power1d=True)
    t0 = time.perf_counter()
    O.sinkhorn_fixed(cost, c.alpha, c.beta, c.eps, c.rho, c.rho, "h", iters)
    el = time.perf_counter() - t0
    return iters / el, 1, f"{iters} H iterations of cfg1 (oracle port, one thread)"


# ---------------------------------------------------------------------------
# Headline: cfg3 TI-Sinkhorn (row-sharded for N > 1).


def cfg3_config(c, world):
    """The config dict of the headline line -- shared with --impl reference so
    both arms name the same workload."""
    return {"workload": "cfg3: H-Sinkhorn N=M=65536 d=2 fp32, eps=1e-2*max|x-y|^2, KL rho=1",
            "n": len(c.x), "m": len(c.y), "d": 2, "eps": c.eps, "rho": c.rho, "variant": "h",
            "parallelism": f"rows/{world} (NCCL all-gather per iteration)" if world > 1
            else "single GPU",
            "iters_per_step": CFG3_ITERS,
            "step": f"one {CFG3_ITERS}-iteration solve from zero potentials (sinkhorn_batched)",
            "l2": f"{L2_FLUSH_BYTES >> 20} MiB write between steps (included in timing)"}


def run_cfg3(args, rank, world, dev, comm):
    import torch

    import paper_2201_00730_b200 as P
    from paper_2201_00730_b200 import _device as D
    from paper_2201_00730_b200 import _lib
    from paper_2201_00730_b200 import synthetic as S
    from paper_2201_00730_b200.distributed import row_offset, shard_rows

    lib = _lib.load()
    c = S.cfg3_inputs()
    n, m = len(c.x), len(c.y)
    rows = shard_rows(n, world)
    off = row_offset(n, world, rank)
    nl = rows[rank]
    xl, al = c.x[off:off + nl], c.alpha[off:off + nl]
    x = torch.as_tensor(xl, dtype=torch.float32, device=dev)
    a = torch.as_tensor(al, dtype=torch.float32, device=dev)
    y = torch.as_tensor(c.y, dtype=torch.float32, device=dev)
    b = torch.as_tensor(c.beta, dtype=torch.float32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    kw = dict(comm=comm.handle, nranks=world, rank=rank) if comm is not None else {}

    def step():
        f, g, _, _ = P.sinkhorn_batched(x, y, a, b, c.eps, c.rho, c.rho, CFG3_ITERS, variant="h",
                                        precision="fp32", **kw)
        return f, g

    for _ in range(max(args.warmup, 3)):
        f, g = step()
    flush.zero_()
    with cuda_timer() as tf:
        flush.zero_()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        with cuda_timer() as tt:
            for _ in range(args.steps):
                flush.zero_()
                f, g = step()
    ms_step = max_over_ranks(tt.ms / args.steps, world, dev)
    value = CFG3_ITERS * 1e3 / ms_step
    # the same workload as one-iteration calls with a flush before every iteration (the
    # step definition used until round 2's last session), for comparison only
    fi = f
    with cuda_timer() as t1:
        for _ in range(20):
            flush.zero_()
            fi, _g, _, _ = P.sinkhorn_batched(x, y, a, b, c.eps, c.rho, c.rho, 1, variant="h",
                                              precision="fp32", f0=fi, **kw)
    ms_call = max_over_ranks(t1.ms / 20, world, dev)

    # roofline of the dominant kernel (fused cost + online LSE half-step),
    # timed live with CUDA events on the launching stream, on this rank's shard.
    f_, g_, tr_, its_ = P.sinkhorn_batched(x, y, a, b, c.eps, c.rho, c.rho, 1, precision="fp32",
                                           f0=f)
    ms2 = (ctypes.c_float * 2)()
    desc = _lib.SinkhornDesc(
        variant=_lib.SINKHORN_H, dtype=_lib.F32, cost=_lib.COST_SQEUCLID, batch=1, n=nl, m=m, d=2,
        p=2.0, eps=c.eps, rho1=c.rho, rho2=c.rho, x=_lib.ptr(x), y=_lib.ptr(y), c=None, ct=None,
        a=_lib.ptr(a), b=_lib.ptr(b), f=_lib.ptr(f_), g=_lib.ptr(g_), init_given=1, iters=1,
        tol=0.0, use_tol=0, trace_delta=_lib.ptr(tr_), iterations=_lib.ptr(its_),
        nccl_comm=None, nranks=1, rank=0, shard_rows=None)
    size = ctypes.c_size_t(0)
    _lib.check(lib.uot_sinkhorn_workspace_size(ctypes.byref(desc), ctypes.byref(size)))
    ws = D.workspace(size.value)
    lib.uot_sinkhorn_time_main.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                           ctypes.c_void_p, ctypes.c_int,
                                           ctypes.POINTER(ctypes.c_float)]
    _lib.check(lib.uot_sinkhorn_time_main(ctypes.byref(desc), _lib.ptr(ws), size.value,
                                          _lib.stream_handle(), 20, ms2))
    kernel_ms = 0.5 * (ms2[0] + ms2[1])
    probes = load_probes()
    live = ctypes.c_double(0.0)
    lib.uot_probe_mufu_ex2.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)]
    _lib.check(lib.uot_probe_mufu_ex2(_lib.stream_handle(), ctypes.byref(live)))
    achieved = float(nl) * float(m) / (kernel_ms * 1e-3) / 1e9
    peak_g = probes["ex2_per_s"] / 1e9

    e2e = run_cfg3_e2e(P, c, xl, al, args.steps, dev, kw, world)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            traffic = json.load(fh)["sk_main_sq2"]["dram_bytes_per_launch"] if world == 1 else None
    except (OSError, KeyError, ValueError):
        traffic = None
    roof = {"bound": "mufu", "achieved": achieved, "peak": peak_g, "unit": "Gex2/s",
            "frac": achieved / peak_g, "traffic": traffic,
            "kernel": "sk_main_sq2", "kernel_ms": kernel_ms,
            "work_per_launch": f"{nl}*{m} ex2",
            "peak_source": probes["source"], "peak_live_probe": live.value / 1e9}
    line = {
        "metric": METRIC, "value": value, "unit": "iter/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded 8-component 2-D Gaussian mixtures, BASELINE cfg3)",
        "config": cfg3_config(c, world), "l2_flush_ms": tf.ms,
        "single_iteration_calls": {"value": 1e3 / ms_call, "unit": "iter/s", "ms_per_call": ms_call,
                                   "note": "20 one-iteration calls, L2 flush before each"},
        "roofline": roof, "e2e": e2e,
        # per iteration: 2 main kernels + 2 tails (+ the combine when sharded), replayed from
        # the captured two-iteration graph; per solve: centre, zero, reset, finalize, ...
        "gpu_launches": ((4 if world == 1 else 5) * CFG3_ITERS + (7 if world == 1 else 8))
        * args.steps,
    }
    return line, clk


def run_cfg3_e2e(P, c, xl, al, steps, dev, kw, world):
    """Same metric through the public API from pinned host buffers: H2D of
    the step's inputs, one CFG3_ITERS-iteration solve, D2H of the resulting
    potentials -- the call a user of the reference's run() makes."""
    import torch

    host = {k: torch.as_tensor(v, dtype=torch.float32).pin_memory()
            for k, v in (("x", xl), ("y", c.y), ("a", al), ("b", c.beta))}
    out_f = torch.empty(len(xl), dtype=torch.float32).pin_memory()
    out_g = torch.empty(len(c.y), dtype=torch.float32).pin_memory()

    def one():
        dv = {k: v.to(dev, non_blocking=True) for k, v in host.items()}
        f, g, _, _ = P.sinkhorn_batched(dv["x"], dv["y"], dv["a"], dv["b"], c.eps, c.rho, c.rho,
                                        CFG3_ITERS, precision="fp32", **kw)
        out_f.copy_(f[0], non_blocking=True)
        out_g.copy_(g[0], non_blocking=False)

    for _ in range(2):
        one()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with cuda_timer() as t:
        for _ in range(steps):
            one()
    ms = max_over_ranks(t.ms / steps, world, dev)
    n, m = len(xl), len(c.y)
    return {"value": CFG3_ITERS * 1e3 / ms, "unit": "iter/s",
            "h2d_bytes_per_step": 4 * (2 * n + 2 * m + n + m),
            "d2h_bytes_per_step": 4 * (n + m), "ms_per_step": ms,
            "path": "paper_2201_00730_b200.sinkhorn_batched -> uot_sinkhorn_run (C-ABI)"}


# ---------------------------------------------------------------------------
# Secondary BASELINE configs (sharded by problem across ranks).


def run_cfg2(rank, world, dev, peaks):
    import torch

    import paper_2201_00730_b200 as P
    from paper_2201_00730_b200 import synthetic as S
    from paper_2201_00730_b200.distributed import shard_problems

    lo, hi = shard_problems(4096, world, rank)
    x, y, a, b = S.cfg2_batch(batch=4096, start=lo, count=hi - lo)
    x, y, a, b = (torch.as_tensor(v, device=dev) for v in (x, y, a, b))
    iters = 500
    # warm-up with the timed shapes, so the caching allocator already holds the
    # trace / workspace blocks (their cudaMalloc is not part of an iteration)
    P.fw_solve_batched(x, y, a, b, 1.0, 1.0, 2.0, iters, "linesearch")
    torch.cuda.synchronize()
    with cuda_timer() as t:
        r = P.fw_solve_batched(x, y, a, b, 1.0, 1.0, 2.0, iters, "linesearch")
    ms = max_over_ranks(t.ms, world, dev)
    assert int(r.status.max().item()) == 0
    it_s = iters / (ms * 1e-3)
    gbs = CFG2_BYTES_PER_ITER * it_s / 1e9
    # the bound that applies (the state is on chip): SM issue slots, from the
    # committed instruction count of the same workload (profiles/r2_cfg2_issue.json)
    issue = None
    try:
        with open(os.path.join(ROOT, "profiles", "r2_cfg2_issue.json")) as fh:
            ipi = json.load(fh)["warp_instr_per_problem_iteration"]
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        peak_i = sms * 4 * 1.965e9 / 1e9  # G warp-instructions/s at the max SM clock
        ach_i = ipi * (hi - lo) * it_s / 1e9
        issue = {"bound": "issue", "achieved": ach_i, "peak": peak_i, "unit": "Gwarp-instr/s",
                 "frac": ach_i / peak_i,
                 "work_per_iteration": f"{ipi} warp-instructions per problem-iteration (ncu, "
                                       "500 line-search iterations)"}
    except (OSError, KeyError, ValueError):
        pass
    return {"workload": "cfg2: batched 1-D FW, B=4096, N=M=1024, KL rho=1, |x-y|^2, fp64, "
                        "500 line-search iterations (fixed count)",
            "issue": issue,
            "value": it_s, "unit": "iter/s (batched FW iterations over all 4096 problems)",
            "ms_total": ms, "dtype": "f64", "scaling": "weak-by-problem" if world > 1 else None,
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": gbs / peaks["hbm_gbs"],
                         "work_per_iteration": "268,435,456 algorithmic bytes (SURVEY.md §8d)",
                         "note": "state resident on chip for all iterations (one CTA per "
                                 "problem): DRAM traffic ~0 per iteration; the kernel is bound "
                                 "by fp64 exp / reductions, see DESIGN.md"}}


def run_cfg2_pfw(rank, world, dev, peaks):
    """§8f row 1: pairwise FW on the cfg2 batch (the atom store lives in HBM;
    every iteration streams the active atoms once for scores and dedup)."""
    import torch

    import paper_2201_00730_b200 as P
    from paper_2201_00730_b200 import synthetic as S
    from paper_2201_00730_b200.distributed import shard_problems

    lo, hi = shard_problems(4096, world, rank)
    x, y, a, b = S.cfg2_batch(batch=4096, start=lo, count=hi - lo)
    x, y, a, b = (torch.as_tensor(v, device=dev) for v in (x, y, a, b))
    iters = 200
    P.fw_solve_batched(x, y, a, b, 1.0, 1.0, 2.0, iters, "pairwise")  # warm-up, same shapes
    torch.cuda.synchronize()
    with cuda_timer() as t:
        r = P.fw_solve_batched(x, y, a, b, 1.0, 1.0, 2.0, iters, "pairwise")
    ms = max_over_ranks(t.ms, world, dev)
    assert int(r.status.max().item()) == 0
    na = r.natoms.double()
    # atom-store bytes per batched iteration: scores + dedup pass over the
    # active atoms (n+m doubles each) + the away-atom row + the new atom row
    rows = float((na.mean(dim=0) + 2.0).mean().item()) * na.shape[0]
    store_bytes = rows * 2048 * 8
    it_s = iters / (ms * 1e-3)
    gbs = store_bytes * it_s / 1e9
    return {"workload": "cfg2 pairwise FW (SURVEY.md 8f row 1): B=4096, N=M=1024, KL rho=1, "
                        f"|x-y|^2, fp64, {iters} pairwise iterations (fixed count)",
            "value": it_s, "unit": "iter/s (batched PFW iterations over all 4096 problems)",
            "ms_total": ms, "dtype": "f64",
            "mean_active_atoms": float(na.mean().item()),
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": gbs / peaks["hbm_gbs"],
                         "work_per_iteration": f"{store_bytes:.3e} atom-store bytes (active atoms "
                                               "+ away + new rows, measured mean)",
                         "note": "the LMO part is the on-chip FW iteration (see cfg2_fw)"}}


def run_cfg5(rank, world, dev, peaks):
    import torch

    import paper_2201_00730_b200 as P
    from paper_2201_00730_b200 import synthetic as S
    from paper_2201_00730_b200.distributed import shard_problems

    lo, hi = shard_problems(64, world, rank)
    xs, ws = S.cfg5_batch(start=lo, count=hi - lo)
    x, a = torch.as_tensor(xs, device=dev), torch.as_tensor(ws, device=dev)
    w = np.full(16, 1 / 16)
    iters = 1000
    P.fw_barycenter_batched(x, a, w, 1.0, iters, "linesearch")  # warm-up, same shapes
    torch.cuda.synchronize()
    with cuda_timer() as t:
        r = P.fw_barycenter_batched(x, a, w, 1.0, iters, "linesearch")
    ms = max_over_ranks(t.ms, world, dev)
    assert int(r.status.max().item()) == 0
    it_s = iters / (ms * 1e-3)
    gbs = CFG5_BYTES_PER_ITER * it_s / 1e9
    return {"workload": "cfg5: barycenter FW, 64 problems x K=16 x N=8192, KL rho=1, fp64, "
                        "1000 line-search iterations (fixed count)",
            "value": it_s, "unit": "iter/s (batched FW iterations over all 64 problems)",
            "ms_total": ms, "dtype": "f64",
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": gbs / peaks["hbm_gbs"],
                         "work_per_iteration": "268,435,456 algorithmic bytes (SURVEY.md §8d)"}}


def run_cfg1(dev):
    import torch

    import paper_2201_00730_b200 as P
    from paper_2201_00730_b200 import synthetic as S

    c = S.cfg1_inputs()
    out = {}
    for v in ("h", "f", "g"):
        P.sinkhorn_batched(c.x[None], c.y[None], c.alpha[None], c.beta[None], c.eps, 1.0, 1.0, 10,
                           variant=v, cost="power", precision="fp64")
        torch.cuda.synchronize()
        with cuda_timer() as t:
            P.sinkhorn_batched(c.x[None], c.y[None], c.alpha[None], c.beta[None], c.eps, 1.0, 1.0,
                               1000, variant=v, cost="power", precision="fp64")
        out[v] = 1000 / (t.ms * 1e-3)
    return {"workload": "cfg1: H, F and G Sinkhorn N=M=256 fp64, 1000 iterations (latency bound)",
            "value": out["h"], "unit": "iter/s (H)", "f_variant_iter_s": out["f"],
            "g_variant_iter_s": out["g"], "dtype": "f64"}


def run_cfg3_verify(dev):
    """§8f row 3: dual objective (eps-term) and stationarity residuals of a
    cfg3 pair at full size, two on-the-fly passes (the reference would need
    a 32 GiB cost matrix)."""
    import torch

    import paper_2201_00730_b200 as P
    from paper_2201_00730_b200 import synthetic as S

    c = S.cfg3_inputs()
    f, g, _, _ = P.sinkhorn_batched(c.x[None], c.y[None], c.alpha[None], c.beta[None], c.eps,
                                    c.rho, c.rho, 20, variant="h", precision="fp32")
    P.verify_batched(c.x[None], c.y[None], c.alpha[None], c.beta[None], f, g, c.eps, c.rho, c.rho,
                     precision="fp32")
    torch.cuda.synchronize()
    with cuda_timer() as t:
        out = P.verify_batched(c.x[None], c.y[None], c.alpha[None], c.beta[None], f, g, c.eps,
                               c.rho, c.rho, precision="fp32")
    o = out[0].cpu().numpy()
    return {"workload": "cfg3 pair after 20 H iterations: eps-term log-sum and both "
                        "stationarity residuals, N=M=65536 d=2 fp32",
            "value": t.ms, "unit": "ms per verification (2 on-the-fly passes)",
            "res_f": float(o[2]), "res_g": float(o[0]), "log_eps_sum": float(o[1])}


def run_cfg4(rank, world, dev):
    import torch

    import paper_2201_00730_b200 as P
    from paper_2201_00730_b200 import synthetic as S
    from paper_2201_00730_b200.distributed import shard_problems

    lo, hi = shard_problems(256, world, rank)
    x, y, a, b = S.cfg4_batch(start=lo, count=hi - lo)
    xt, yt, at, bt = (torch.as_tensor(v, dtype=torch.float32, device=dev) for v in (x, y, a, b))
    iters = 300  # the whole BASELINE config-4 solve
    P.sinkhorn_batched(xt, yt, at, bt, S.CFG4_EPS, S.CFG4_RHO, S.CFG4_RHO, iters,
                       precision="fp32")  # warm-up, same shapes
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk4:  # tensor + MUFU load: the power cap sets the clock
        with cuda_timer() as t:
            P.sinkhorn_batched(xt, yt, at, bt, S.CFG4_EPS, S.CFG4_RHO, S.CFG4_RHO, iters,
                               precision="fp32")
    ms = max_over_ranks(t.ms, world, dev)
    value = iters / (ms * 1e-3)  # batched iterations over all 256 problems (all ranks)
    # Per 256 x 128 pair tile: 12 kind::f16 MMAs (fp16 hi/lo splits, K = 16)
    # and one kind::tf32 MMA (the row / column constants, K = 8); one ex2 per
    # pair on the MUFU pipe, which now bounds the kernel.
    tiles = 2.0 * 256 * (4096 / 256) * (4096 / 128)  # per iteration (two half-steps)
    tflops = tiles * (12 * 2 * 256 * 128 * 16 + 2 * 256 * 128 * 8) * value / 1e12
    exps = 2.0 * 256 * 4096 * 4096 * value / 1e9
    probes = load_probes()
    peak_g = probes["ex2_per_s"] / 1e9
    peaks, _ = load_peaks()
    # the dominant kernel alone (sk_main_tc, both half-step directions), CUDA
    # events on the launching stream, this rank's shard
    kernel = None
    if world == 1:
        import ctypes

        from paper_2201_00730_b200 import _device as D
        from paper_2201_00730_b200 import _lib

        lib = _lib.load()
        f_, g_, tr_, its_ = P.sinkhorn_batched(xt, yt, at, bt, S.CFG4_EPS, S.CFG4_RHO, S.CFG4_RHO,
                                               1, precision="fp32")
        nb, n4, d4 = xt.shape
        desc = _lib.SinkhornDesc(
            variant=_lib.SINKHORN_H, dtype=_lib.F32, cost=_lib.COST_SQEUCLID, batch=nb, n=n4,
            m=yt.shape[1], d=d4, p=2.0, eps=S.CFG4_EPS, rho1=S.CFG4_RHO, rho2=S.CFG4_RHO,
            x=_lib.ptr(xt), y=_lib.ptr(yt), c=None, ct=None, a=_lib.ptr(at), b=_lib.ptr(bt),
            f=_lib.ptr(f_), g=_lib.ptr(g_), init_given=1, iters=1, tol=0.0, use_tol=0,
            trace_delta=_lib.ptr(tr_), iterations=_lib.ptr(its_), nccl_comm=None, nranks=1,
            rank=0, shard_rows=None)
        size = ctypes.c_size_t(0)
        _lib.check(lib.uot_sinkhorn_workspace_size(ctypes.byref(desc), ctypes.byref(size)))
        ws = D.workspace(size.value)
        ms2 = (ctypes.c_float * 2)()
        lib.uot_sinkhorn_time_main.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                               ctypes.c_void_p, ctypes.c_int,
                                               ctypes.POINTER(ctypes.c_float)]
        _lib.check(lib.uot_sinkhorn_time_main(ctypes.byref(desc), _lib.ptr(ws), size.value,
                                              _lib.stream_handle(), 10, ms2))
        kms = 0.5 * (ms2[0] + ms2[1])
        kach = float(nb) * n4 * yt.shape[1] / (kms * 1e-3) / 1e9
        kernel = {"kernel": "sk_main_tc", "kernel_ms": kms, "achieved": kach,
                  "frac": kach / peak_g,
                  "share_of_iteration": 2.0 * kms / (1e3 / value)}
    c4 = clk4.summary()
    return {"workload": "cfg4: batched H-Sinkhorn B=256 N=M=4096 d=64 fp32, tcgen05 cost tiles "
                        "(kind::f16 hi/lo splits + one kind::tf32 constants MMA, A in TMEM, B "
                        "ring in smem, CTA pairs) + MUFU LSE epilogue; "
                        f"one whole {iters}-iteration solve timed",
            "value": value, "unit": "iter/s", "dtype": "f32 (fp16-split tensor, fp32 accumulate)",
            "clocks": c4,
            "roofline": {"bound": "mufu", "achieved": kernel["achieved"] if kernel else exps,
                         "peak": peak_g, "unit": "Gex2/s",
                         "frac": (kernel["achieved"] if kernel else exps) / peak_g,
                         "kernel": "sk_main_tc" if kernel else None,
                         "kernel_ms": kernel["kernel_ms"] if kernel else None,
                         "work_per_launch": "B*N*M = 4.29e9 ex2",
                         "iteration_frac": exps / peak_g,
                         # the MUFU peak scales with the SM clock; under this kernel's
                         # tensor + MUFU load the power cap holds the clock below its maximum
                         "iteration_frac_at_sampled_clock": (
                             exps / peak_g * c4["sm_max_mhz"] / c4["sm_mhz"]
                             if c4.get("sm_mhz") and c4.get("sm_max_mhz") else None),
                         "kernel_share_of_iteration": kernel["share_of_iteration"] if kernel
                         else None,
                         "peak_source": probes["source"]},
            "tensor": {"achieved_tflops": tflops, "peak_tflops": peaks["bf16_tflops"],
                       "frac": tflops / peaks["bf16_tflops"],
                       "peak_sustained_tflops": peaks.get("bf16_tflops_sustained"),
                       "frac_sustained": tflops / peaks["bf16_tflops_sustained"]
                       if peaks.get("bf16_tflops_sustained") else None,
                       "peak_source": "MEASURED_PEAKS.json dense bf16 (burst / sustained); "
                                      "the fp16 MMAs issue at the bf16 rate"}}


# ---------------------------------------------------------------------------


def run_reference(args, rank, world):
    """--impl reference: the reference's algorithm (the oracle port of
    sinkhorn.py:93-100 / entropies.py:84-92 in C, every host thread) on the
    headline workload.  Each step is the same bounded sample as the headline
    line's cpu_baseline (one g half-step over CFG3_SAMPLE_COLS of the 65536
    columns); value extrapolates it to whole iterations/s.  ms_per_step is the
    measured wall time of one sampled step."""
    if rank != 0:
        return
    from paper_2201_00730_b200 import synthetic as S

    c = S.cfg3_inputs()
    vals, secs = [], []
    for k in range(args.warmup + args.steps):
        v, threads, sample = cpu_cfg3(c)
        if k >= args.warmup:
            vals.append(v)
            secs.append(cpu_cfg3.last_seconds)
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "iter/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * float(np.mean(secs)), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg3_config(c, args.gpus),
        "cpu_baseline": {"value": value, "unit": "iter/s", "cores": threads, "kind": "port",
                         "sample": sample, "value_spread": [float(min(vals)), float(max(vals))]},
        "e2e": {"value": value, "unit": "iter/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "note": "ms_per_step = wall time of one sampled step (not of a whole iteration); value "
                "= the sample's pair rate extrapolated to 2*N*M pairs per iteration",
    }
    print(json.dumps(line), flush=True)


def spawn_ranks(n):
    """--gpus N without torchrun: relaunch this script under
    torch.distributed.run with N local ranks (the driver's own launch line)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def compact(entry):
    """Secondary entries in the printed line: the numbers only (the driver
    keeps a bounded tail of stdout); the descriptive keys go to
    gpurun_out/bench_detail.json."""
    keep = ("value", "unit", "ms_total", "dtype", "f_variant_iter_s", "g_variant_iter_s",
            "mean_active_atoms", "res_f", "res_g", "clocks")
    out = {k: entry[k] for k in keep if k in entry}
    for sub in ("roofline", "tensor", "issue"):
        if entry.get(sub):
            out[sub] = {k: v for k, v in entry[sub].items()
                        if k in ("bound", "achieved", "peak", "unit", "frac", "achieved_tflops",
                                 "peak_tflops", "peak_sustained_tflops", "frac_sustained",
                                 "iteration_frac", "iteration_frac_at_sampled_clock", "kernel")}
    if "cpu_baseline" in entry:
        cb = entry["cpu_baseline"]
        out["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind")}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-secondary", action="store_true")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    comm = None
    if world > 1:
        torch.distributed.init_process_group("nccl", device_id=dev)
        from paper_2201_00730_b200.distributed import NcclComm

        comm = NcclComm(world, rank)
    try:
        peaks, peak_src = load_peaks()
        line, clk = run_cfg3(args, rank, world, dev, comm)
        secondary = {}
        if not args.no_secondary:
            secondary["cfg2_fw"] = run_cfg2(rank, world, dev, peaks)
            secondary["cfg2_pfw"] = run_cfg2_pfw(rank, world, dev, peaks)
            secondary["cfg5_barycenter"] = run_cfg5(rank, world, dev, peaks)
            secondary["cfg4_sinkhorn_d64"] = run_cfg4(rank, world, dev)
            if rank == 0:
                secondary["cfg1_sinkhorn_1d"] = run_cfg1(dev)
                secondary["cfg3_verify"] = run_cfg3_verify(dev)
        if rank == 0:
            cpu_runs = [cpu_cfg3(S_inputs_cfg3()) for _ in range(3)]
            cpu_v = float(np.mean([r_[0] for r_ in cpu_runs]))
            cpu_cores, cpu_sample = cpu_runs[0][1], cpu_runs[0][2] + " (mean of 3 samples)"
            line["cpu_baseline"] = {"value": cpu_v, "unit": "iter/s", "cores": cpu_cores,
                                    "kind": "port", "sample": cpu_sample}
            if not args.no_secondary and world == 1:
                v2, c2, s2 = cpu_cfg2()
                secondary["cfg2_fw"]["cpu_baseline"] = {"value": v2, "unit": "iter/s",
                                                        "cores": c2, "kind": "port", "sample": s2}
                v5, c5, s5 = cpu_cfg5()
                secondary["cfg5_barycenter"]["cpu_baseline"] = {
                    "value": v5, "unit": "iter/s", "cores": c5, "kind": "port", "sample": s5}
                v4, c4, s4 = cpu_cfg4()
                secondary["cfg4_sinkhorn_d64"]["cpu_baseline"] = {
                    "value": v4, "unit": "iter/s", "cores": c4, "kind": "port", "sample": s4}
                v1, c1, s1 = cpu_cfg1()
                secondary["cfg1_sinkhorn_1d"]["cpu_baseline"] = {
                    "value": v1, "unit": "iter/s (H)", "cores": c1, "kind": "port", "sample": s1}
                os.environ["ORACLE_THREADS"] = str(host_cores())
            line["peaks"] = {"hbm_gbs": peaks.get("hbm_gbs"), "source": peak_src}
            line["clocks"] = clk.summary()
            try:
                os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
                with open(os.path.join(ROOT, "gpurun_out", "bench_detail.json"), "w") as fh:
                    json.dump(dict(line, secondary=secondary), fh, indent=1)
            except OSError:
                pass
            line["secondary"] = {k: compact(v) for k, v in secondary.items()}
            print(json.dumps(line), flush=True)
    finally:
        if comm is not None:
            comm.close()
        if world > 1:
            torch.distributed.destroy_process_group()


_CFG3 = None


def S_inputs_cfg3():
    global _CFG3
    if _CFG3 is None:
        from paper_2201_00730_b200 import synthetic as S

        _CFG3 = S.cfg3_inputs()
    return _CFG3


if __name__ == "__main__":
    main()
