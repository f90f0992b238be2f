"""One FW launch (B problems of cfg2 shape, T iterations) for ncu."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2201_00730_b200 as P
from paper_2201_00730_b200 import synthetic as S
B = int(sys.argv[1]) if len(sys.argv) > 1 else 296
T = int(sys.argv[2]) if len(sys.argv) > 2 else 20
step = sys.argv[3] if len(sys.argv) > 3 else "linesearch"
x, y, a, b = S.cfg2_batch(batch=4096, count=B)
dev = torch.device("cuda")
x, y, a, b = (torch.as_tensor(v, device=dev) for v in (x, y, a, b))
r = P.fw_solve_batched(x, y, a, b, 1.0, 1.0, 2.0, T, step)
torch.cuda.synchronize()
print("ok", int(r.iterations[0].item()))
