"""Benchmark driver (contract: see the task README / DESIGN.md §Measurement).

Default workload = BASELINE.json's headline metric quoted on config 3:
TI-Sinkhorn (H variant) on two seeded 8-component 2-D Gaussian mixtures,
N = M = 65536, fp32 log-domain, eps = 1e-2 * max|x - y|^2, KL rho = 1.
A "step" is one full H-Sinkhorn iteration (g half-step + f half-step) over
the whole problem; value = iterations/s of the whole job.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun (N > 1) the single problem is row-sharded across ranks (one
NCCL all-gather of per-column log-sum-exp partials per iteration) and the
step time is the max over ranks of the device-timed step.
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


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "fallback": True}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        time.sleep(0.25)
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
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[5 + k] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port (C, fp64) of the reference's column softmin
# (src/sinkhorn.py:93-100 over src/entropies.py:84-92) on a bounded sample.


def cpu_sinkhorn_rate(c, cols=512):
    import oracle as O

    threads = len(os.sched_getaffinity(0))
    os.environ["ORACLE_THREADS"] = str(threads)
    rng = np.random.default_rng(1)
    sel = np.sort(rng.choice(len(c.y), cols, replace=False))
    cost = O.PointCost(c.x, c.y[sel])
    f = np.zeros(len(c.x))
    t0 = time.perf_counter()
    cost.smin_cols(f, c.eps, c.alpha)
    el = time.perf_counter() - t0
    pairs = len(c.x) * cols
    s_per_iter = el / pairs * 2.0 * len(c.x) * len(c.y)
    sample = (f"one g half-step restricted to {cols} of {len(c.y)} columns x {len(c.x)} rows "
              f"({pairs:.3g} pair evaluations, fp64 C oracle, {threads} threads), "
              f"extrapolated to 2*N*M pairs per iteration")
    return 1.0 / s_per_iter, threads, sample, el


# ---------------------------------------------------------------------------


def run_reference(args, rank, world):
    """--impl reference: the reference's algorithm (oracle port) on host cores."""
    if rank != 0:
        return
    from paper_2201_00730_b200 import synthetic as S

    c = S.cfg3_inputs()
    vals = []
    for k in range(args.warmup + args.steps):
        v, threads, sample, _ = cpu_sinkhorn_rate(c, cols=256)
        if k >= args.warmup:
            vals.append(v)
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "iter/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 / value, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg3: H-Sinkhorn N=M=65536 d=2, eps=1e-2*max|x-y|^2, KL rho=1",
                   "n": len(c.x), "m": len(c.y), "eps": c.eps},
        "cpu_baseline": {"value": value, "unit": "iter/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "iter/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world):
    import torch

    import paper_2201_00730_b200 as P
    from paper_2201_00730_b200 import _device as D
    from paper_2201_00730_b200 import _lib
    from paper_2201_00730_b200 import synthetic as S

    lib = _lib.load()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    c = S.cfg3_inputs()
    n, m = len(c.x), len(c.y)
    x = torch.as_tensor(c.x, dtype=torch.float32, device=dev)
    y = torch.as_tensor(c.y, dtype=torch.float32, device=dev)
    a = torch.as_tensor(c.alpha, dtype=torch.float32, device=dev)
    b = torch.as_tensor(c.beta, dtype=torch.float32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def step(f0):
        f, g, _, _ = P.sinkhorn_batched(x, y, a, b, c.eps, c.rho, c.rho, 1, variant="h",
                                        precision="fp32", f0=f0)
        return f, g

    # warm-up (also builds the first potentials)
    f = None
    for _ in range(max(args.warmup, 3)):
        f, g = step(f)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    flush_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    # time the L2 flush alone so it can be reported (it is included below)
    flush_ev[0].record(st)
    flush.zero_()
    flush_ev[1].record(st)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        e0.record(st)
        for _ in range(args.steps):
            flush.zero_()
            f, g = step(f)
        e1.record(st)
        torch.cuda.synchronize()
    ms_total = e0.elapsed_time(e1)
    flush_ms = flush_ev[0].elapsed_time(flush_ev[1])
    ms_step = ms_total / args.steps
    if world > 1:
        tt = torch.tensor([ms_step], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms_step = float(tt.item())
    value = 1e3 / ms_step

    # roofline of the dominant kernel: the fused log-sum-exp half-step
    desc_f, desc_g, its = None, None, None
    f_, g_, tr_, its_ = P.sinkhorn_batched(x, y, a, b, c.eps, c.rho, c.rho, 1, precision="fp32",
                                           f0=f)
    ms2 = (ctypes.c_float * 2)()
    desc = _lib.SinkhornDesc(
        variant=_lib.SINKHORN_H, dtype=_lib.F32, cost=_lib.COST_SQEUCLID, batch=1, n=n, m=m, d=2,
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
    ex2_per_launch = float(n) * float(m)
    peak = ctypes.c_double(0.0)
    lib.uot_probe_mufu_ex2.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)]
    _lib.check(lib.uot_probe_mufu_ex2(_lib.stream_handle(), ctypes.byref(peak)))
    achieved = ex2_per_launch / (kernel_ms * 1e-3) / 1e9
    peak_g = peak.value / 1e9

    # end-to-end through the public API with host buffers each step
    e2e = run_e2e(P, c, args.steps, dev)

    if rank != 0:
        return
    cpu_v, cpu_threads, cpu_sample, _ = cpu_sinkhorn_rate(c)
    launches_per_step = 4 + 6  # 2x(main+tail) + reset, 3x zero, init tail, finalize per call
    line = {
        "metric": METRIC, "value": value, "unit": "iter/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded 8-component 2-D Gaussian mixtures, BASELINE cfg3)",
        "config": {
            "workload": "cfg3: H-Sinkhorn N=M=65536 d=2 fp32, eps=1e-2*max|x-y|^2, KL rho=1",
            "n": n, "m": m, "d": 2, "eps": c.eps, "rho": c.rho, "variant": "h",
            "parallelism": f"rows/{world}" if world > 1 else "single",
            "l2": f"{L2_FLUSH_BYTES >> 20} MiB write between steps (included; "
                  f"{flush_ms:.3f} ms each)",
        },
        "roofline": {"bound": "mufu", "achieved": achieved, "peak": peak_g, "unit": "Gex2/s",
                     "frac": achieved / peak_g, "traffic": None,
                     "kernel": "sk_main<SqE32<2>> (fused cost + online LSE half-step)",
                     "kernel_ms": kernel_ms, "work_per_launch": f"{n}*{m} ex2",
                     "peak_source": "measured live: uot_probe_mufu_ex2 (all SMs, CUDA events)"},
        "cpu_baseline": {"value": cpu_v, "unit": "iter/s", "cores": cpu_threads, "kind": "port",
                         "sample": cpu_sample},
        "e2e": e2e,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def run_e2e(P, c, steps, dev):
    """Same metric through the public API from pinned host buffers: H2D of
    the step's inputs, one iteration, D2H of the resulting pair."""
    import torch

    n, m = len(c.x), len(c.y)
    host = {k: torch.as_tensor(v, dtype=torch.float32).pin_memory()
            for k, v in (("x", c.x), ("y", c.y), ("a", c.alpha), ("b", c.beta))}
    fh = torch.zeros(n, dtype=torch.float32).pin_memory()
    out_f = torch.empty(n, dtype=torch.float32).pin_memory()
    out_g = torch.empty(m, dtype=torch.float32).pin_memory()
    st = torch.cuda.current_stream()

    def one():
        dv = {k: v.to(dev, non_blocking=True) for k, v in host.items()}
        f0 = fh.to(dev, non_blocking=True)
        f, g, _, _ = P.sinkhorn_batched(dv["x"], dv["y"], dv["a"], dv["b"], c.eps, c.rho, c.rho,
                                        1, precision="fp32", f0=f0)
        out_f.copy_(f[0], non_blocking=True)
        out_g.copy_(g[0], non_blocking=True)
        fh.copy_(out_f)

    for _ in range(2):
        one()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        one()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    h2d = 4 * (2 * n + 2 * m + n + m + n)
    d2h = 4 * (n + m)
    return {"value": 1e3 / ms, "unit": "iter/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        torch.distributed.init_process_group("nccl")
    try:
        run_ours(args, rank, world)
    finally:
        if world > 1:
            import torch

            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
