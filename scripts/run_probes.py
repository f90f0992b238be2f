"""Measure the roofline denominators MEASURED_PEAKS.json does not carry --
MUFU ex2.approx.f32 and FP64 DFMA throughput -- with the SM clock sampled
during the probes, and write them to profiles/r2_probes.json.  bench.py uses
the committed figures as FIXED denominators (the live probe made
the denominator vary from box to box).

    python scripts/run_probes.py [--out profiles/r2_probes.json]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_probes.json"))
    ap.add_argument("--reps", type=int, default=15)
    args = ap.parse_args()
    import torch

    from bench import ClockSampler
    from paper_2201_00730_b200 import _lib

    lib = _lib.load()
    torch.cuda.set_device(0)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    dp = ctypes.POINTER(ctypes.c_double)
    lib.uot_probe_mufu_ex2.argtypes = [ctypes.c_void_p, dp]
    lib.uot_probe_dfma.argtypes = [ctypes.c_void_p, dp]
    out = {"sms": sms, "device": torch.cuda.get_device_name(0)}
    for name, fn in (("ex2", lib.uot_probe_mufu_ex2), ("dfma", lib.uot_probe_dfma)):
        vals = []
        with ClockSampler(0) as clk:
            for _ in range(args.reps):
                v = ctypes.c_double(0.0)
                _lib.check(fn(_lib.stream_handle(), ctypes.byref(v)))
                vals.append(v.value)
        c = clk.summary()
        med = float(np.median(vals))
        mhz = c["sm_mhz"] or c["sm_max_mhz"]
        per_clk = med / (sms * mhz * 1e6) if mhz else None
        out[name] = {"per_s_median": med, "per_s_max": float(max(vals)),
                     "per_s_min": float(min(vals)), "clocks": c,
                     "per_clk_per_sm": per_clk,
                     "per_s_at_max_clock": per_clk * sms * c["sm_max_mhz"] * 1e6
                     if per_clk and c["sm_max_mhz"] else None}
    out["note"] = ("ex2: uot_probe_mufu_ex2 (8 independent ex2.approx.ftz.f32 chains per thread, "
                   "8 CTAs of 256 threads per SM); dfma: uot_probe_dfma (8 independent DFMA "
                   "chains per thread); CUDA events; clocks sampled by nvidia-smi every 100 ms")
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
