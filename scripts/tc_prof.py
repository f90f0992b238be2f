"""Wait-cycle breakdown of sk_main_tc (needs the -DUOT_TC_PROF build)."""
import os, sys, ctypes
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2201_00730_b200 as P
from paper_2201_00730_b200 import synthetic as S
from paper_2201_00730_b200 import _lib
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
x, y, a, b = S.cfg4_batch(count=B)
xt, yt, at, bt = (torch.as_tensor(v, dtype=torch.float32, device="cuda") for v in (x, y, a, b))
lib = _lib.load()
buf = (ctypes.c_ulonglong * 8)()
P.sinkhorn_batched(xt, yt, at, bt, S.CFG4_EPS, S.CFG4_RHO, S.CFG4_RHO, 1, precision="fp32")
torch.cuda.synchronize()
lib.uot_tc_prof(buf, 1)
P.sinkhorn_batched(xt, yt, at, bt, S.CFG4_EPS, S.CFG4_RHO, S.CFG4_RHO, 4, precision="fp32")
torch.cuda.synchronize()
lib.uot_tc_prof(buf, 1)
names = ["prod wait empty", "mma wait full", "mma wait dempty", "epi wait dfull (per warp)",
         "prologue", "total", "epi math", "mma issue"]
ctas = 2 * 4 * B * 32
for i, nme in enumerate(names):
    print(f"{nme:28s} {buf[i] / ctas:12.0f} cycles/CTA")
