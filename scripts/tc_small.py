import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2201_00730_b200 as P
from paper_2201_00730_b200 import synthetic as S
n, m, d = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
x, y, a, b = S.cfg4_batch(batch=2, n=n, m=m, d=d)
f, g, _, _ = P.sinkhorn_batched(x, y, a, b, S.CFG4_EPS, S.CFG4_RHO, S.CFG4_RHO, 3, precision="fp32")
torch.cuda.synchronize()
print("ok", n, m, d, float(f.abs().max()), flush=True)
