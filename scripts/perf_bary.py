"""Time batched barycenter FW on cfg5 (64 x K=16 x N=8192)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2201_00730_b200 as P
from paper_2201_00730_b200 import synthetic as S
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
t0 = time.time(); xs, ws = S.cfg5_batch(count=B); print(f"gen {time.time()-t0:.1f}s", flush=True)
dev = torch.device("cuda")
x = torch.as_tensor(xs, device=dev); a = torch.as_tensor(ws, device=dev)
w = np.full(16, 1 / 16)
for iters in (2, 22):
    r = P.fw_barycenter_batched(x, a, w, 1.0, iters, "linesearch")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    r = P.fw_barycenter_batched(x, a, w, 1.0, iters, "linesearch")
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"iters={iters}: {ms:.2f} ms, wall {1e3*(time.perf_counter()-t1):.1f} ms, status {r.status.max().item()}", flush=True)
