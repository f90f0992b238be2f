"""Per-CTA timeline of sk_main_tc (timing build: UOT_B200_VARIANT=tct
UOT_NVCC_EXTRA=-DUOT_TC_TIMING): prologue, fill (first tile), steady state,
drain, as averages over the CTAs of one cfg4 half-step (64 problems)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2201_00730_b200 as P
from paper_2201_00730_b200 import _lib
from paper_2201_00730_b200 import synthetic as S
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
x, y, a, b = S.cfg4_batch(count=B)
xt, yt, at, bt = (torch.as_tensor(v, dtype=torch.float32, device="cuda") for v in (x, y, a, b))
P.sinkhorn_batched(xt, yt, at, bt, S.CFG4_EPS, S.CFG4_RHO, S.CFG4_RHO, 1, precision="fp32")
torch.cuda.synchronize()
lib = _lib.load()
n = B * 16  # CTAs of one launch (two 128-row blocks per CTA, 4096 outputs)
buf = (ctypes.c_ulonglong * (8 * n))()
lib.uot_debug_tc_stamps(buf, n)
t8 = np.array(buf, dtype=np.float64).reshape(n, 8)
t8 = t8[t8[:, 0] > 0]
t = t8[:, :5]
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
d = np.diff(t, axis=1) / 1e3
print(f"CTAs {len(t)}; span {(t[:, 4].max() - t0) / 1e3:.1f} us")
for k, name in enumerate(["prologue", "fill (first tile)", "tiles", "drain"]):
    print(f"{name:18s} mean {d[:, k].mean():7.2f} us  p10 {np.percentile(d[:, k], 10):7.2f}  p90 {np.percentile(d[:, k], 90):7.2f}")
life = (t[:, 4] - t[:, 0]) / 1e3
print(f"lifetime mean {life.mean():.2f} us; concurrent CTAs ~ {life.sum() / ((t[:, 4].max() - t0) / 1e3):.1f}")
sub = t8[:, [0, 5, 6, 7, 1]]
for k, name in enumerate(["alloc + barrier init", "stage outputs", "build A in TMEM", "cluster sync"]):
    dd = np.diff(sub, axis=1)[:, k] / 1e3
    print(f"  prologue: {name:22s} mean {dd.mean():7.2f} us")
