"""Average Newton passes per line search for cfg2 FW and cfg5 barycenter.
Needs the stats build: UOT_B200_VARIANT=stats UOT_NVCC_EXTRA=-DUOT_NEWTON_STATS
python -m paper_2201_00730_b200.build, then UOT_B200_LIB=.../_uot_b200_stats.so."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2201_00730_b200 as P
from paper_2201_00730_b200 import _lib
from paper_2201_00730_b200 import synthetic as S
lib = _lib.load()
buf = (ctypes.c_ulonglong * 2)()
dev = torch.device("cuda")
x, y, a, b = (torch.as_tensor(v, device=dev) for v in S.cfg2_batch(batch=512))
for iters in (20, 200):
    lib.uot_debug_fw_stats(buf, 1)
    P.fw_solve_batched(x, y, a, b, 1.0, 1.0, 2.0, iters, "linesearch")
    torch.cuda.synchronize()
    lib.uot_debug_fw_stats(buf, 1)
    print(f"cfg2 FW {iters} its: {buf[0] / max(buf[1], 1):.2f} passes per line search "
          f"({buf[1]} searches)")
xs, ws = S.cfg5_batch(count=16)
xt, at = torch.as_tensor(xs, device=dev), torch.as_tensor(ws, device=dev)
for iters in (20, 100):
    lib.uot_debug_mot_stats(buf, 1)
    P.fw_barycenter_batched(xt, at, np.full(16, 1 / 16), 1.0, iters, "linesearch")
    torch.cuda.synchronize()
    lib.uot_debug_mot_stats(buf, 1)
    print(f"cfg5 bary {iters} its: {buf[0] / max(buf[1], 1):.2f} passes per line search "
          f"({buf[1]} searches)")
