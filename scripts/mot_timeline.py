"""Phase timeline of mot_update (timing build: UOT_B200_VARIANT=mtt
UOT_NVCC_EXTRA=-DUOT_MOT_TIMING): load, scan + gap sums, cluster sums,
line search, update, log-sum-exp, tilt, final cluster sync -- averaged over
the CTAs of the last update launch of a short cfg5 run."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2201_00730_b200 as P
from paper_2201_00730_b200 import _lib
from paper_2201_00730_b200 import synthetic as S
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
xs, ws = S.cfg5_batch(count=B)
dev = torch.device("cuda")
P.fw_barycenter_batched(torch.as_tensor(xs, device=dev), torch.as_tensor(ws, device=dev),
                        np.full(16, 1 / 16), 1.0, 3, "linesearch")
torch.cuda.synchronize()
lib = _lib.load()
n = B * 16
buf = (ctypes.c_ulonglong * (8 * n))()
lib.uot_debug_mot_stamps(buf, n)
t = np.array(buf, dtype=np.float64).reshape(n, 8)
t = t[t[:, 0] > 0]
d = np.diff(t, axis=1) / 1e3
names = ["load dcc/f/ta/a", "scan + gap sums", "cluster sum + scalars", "line search",
         "update + store", "log-sum-exp", "tilt + samples", "cluster sync"]
if os.environ.get("UOT_MOT_UPDATE1") != "1":  # mot_update2 phases
    names = ["load rows", "scan + gap sums", "cluster sum", "line search",
             "update + LSE + drain", "tilt x2 + samples", "cluster sync"]
for k in range(len(names)):
    print(f"{names[k]:24s} mean {d[:, k].mean():7.2f} us  p90 {np.percentile(d[:, k], 90):7.2f}")
life = (t[:, 7] - t[:, 0]) / 1e3
print(f"CTA lifetime mean {life.mean():.2f} us; span {(t[:, 7].max() - t[:, 0].min()) / 1e3:.1f} us")
