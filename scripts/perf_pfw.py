"""Time batched pairwise FW on cfg2 (B=4096, N=M=1024, 200 iterations)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2201_00730_b200 as P
from paper_2201_00730_b200 import synthetic as S
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
x, y, a, b = S.cfg2_batch(batch=B)
dev = torch.device("cuda")
x, y, a, b = (torch.as_tensor(v, device=dev) for v in (x, y, a, b))
for rep in range(2):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    r = P.fw_solve_batched(x, y, a, b, 1.0, 1.0, 2.0, iters, "pairwise")
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
print(f"pairwise iters={iters}: {ms:.2f} ms total, {ms/iters*1e3:.1f} us/iter, {iters/ms*1e3:.0f} iter/s; "
      f"status {int(r.status.max())}, mean atoms {float(r.natoms[:, -1].float().mean()):.2f}, "
      f"h0[-1] mean {float(r.h0[:, -1].mean()):.12f}")
