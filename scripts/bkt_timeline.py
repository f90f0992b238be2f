"""Phase timeline of mot_bucket (timing build: UOT_B200_VARIANT=mtt
UOT_NVCC_EXTRA=-DUOT_MOT_TIMING): prologue, gather, sort, scan, store."""
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
                        np.full(16, 1 / 16), 1.0, 1, "linesearch")
torch.cuda.synchronize()
lib = _lib.load()
n = 1 << 14
buf = (ctypes.c_ulonglong * (6 * n))()
lib.uot_debug_bkt_stamps(buf, n)
t = np.array(buf, dtype=np.float64).reshape(n, 6)[:, :5]
t = t[t[:, 0] > 0]
d = np.diff(t, axis=1) / 1e3
for k, nm in enumerate(["prologue", "gather", "sort", "scan", "store"][:d.shape[1]]):
    print(f"{nm:10s} mean {d[:, k].mean():7.2f} us  p90 {np.percentile(d[:, k], 90):7.2f}")
life = (t[:, 4] - t[:, 0]) / 1e3
print(f"CTAs {len(t)}; lifetime mean {life.mean():.2f} us; span {(t[:, 4].max() - t[:, 0].min()) / 1e3:.1f} us")
