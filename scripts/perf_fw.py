"""Time batched FW on cfg2 (B=4096, N=M=1024) for a few iteration counts."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2201_00730_b200 as P
from paper_2201_00730_b200 import synthetic as S
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
t0 = time.time()
x, y, a, b = S.cfg2_batch(batch=B)
print(f"gen {time.time()-t0:.1f}s", flush=True)
dev = torch.device("cuda")
x, y, a, b = (torch.as_tensor(v, device=dev) for v in (x, y, a, b))
for iters in (5, 50):
    r = P.fw_solve_batched(x, y, a, b, 1.0, 1.0, 2.0, iters, "linesearch")
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    r = P.fw_solve_batched(x, y, a, b, 1.0, 1.0, 2.0, iters, "linesearch")
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"linesearch iters={iters}: {ms:.2f} ms total, {ms/iters*1e3:.1f} us/iter, {iters/ms*1e3:.0f} iter/s, "
          f"alg GB/s {268435456*iters/(ms*1e-3)/1e9:.0f}", flush=True)
    rh = P.fw_solve_batched(x, y, a, b, 1.0, 1.0, 2.0, iters, "harmonic")
    torch.cuda.synchronize(); e0.record()
    rh = P.fw_solve_batched(x, y, a, b, 1.0, 1.0, 2.0, iters, "harmonic")
    e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1)
    print(f"harmonic   iters={iters}: {ms:.2f} ms total, {ms/iters*1e3:.1f} us/iter", flush=True)
