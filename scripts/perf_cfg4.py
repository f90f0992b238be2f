import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, ctypes
import paper_2201_00730_b200 as P
from paper_2201_00730_b200 import synthetic as S
B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
t0 = time.time(); x, y, a, b = S.cfg4_batch(count=B); print(f"gen {time.time()-t0:.1f}s", flush=True)
xt, yt, at, bt = (torch.as_tensor(v, dtype=torch.float32, device="cuda") for v in (x, y, a, b))
for iters in (2, 12):
    P.sinkhorn_batched(xt, yt, at, bt, S.CFG4_EPS, S.CFG4_RHO, S.CFG4_RHO, iters, precision="fp32")
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    P.sinkhorn_batched(xt, yt, at, bt, S.CFG4_EPS, S.CFG4_RHO, S.CFG4_RHO, iters, precision="fp32")
    e1.record(); torch.cuda.synchronize()
    print(f"iters={iters}: {e0.elapsed_time(e1):.2f} ms", flush=True)
