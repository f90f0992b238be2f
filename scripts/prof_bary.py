"""A short cfg5 barycenter FW run (B problems, T iterations) for ncu."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2201_00730_b200 as P
from paper_2201_00730_b200 import synthetic as S
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
T = int(sys.argv[2]) if len(sys.argv) > 2 else 3
xs, ws = S.cfg5_batch(count=B)
dev = torch.device("cuda")
x = torch.as_tensor(xs, device=dev); a = torch.as_tensor(ws, device=dev)
r = P.fw_barycenter_batched(x, a, np.full(16, 1 / 16), 1.0, T, "linesearch")
torch.cuda.synchronize()
print("ok", int(r.status.max().item()))
