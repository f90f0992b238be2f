"""Per-iteration time of one FW problem (and a batch of 148) at sizes around the
resident / large-problem boundary."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2201_00730_b200 as P
from paper_2201_00730_b200 import synthetic as S
dev = torch.device("cuda")
for n in (1024, 4096, 4100, 5000, 8192, 16384):
    for B in (1, 148):
        x, y, a, b = S.cfg2_batch(batch=B, n=n, m=n, seed=3)
        x, y, a, b = (torch.as_tensor(v, device=dev) for v in (x, y, a, b))
        out = []
        for iters in (10, 60):
            P.fw_solve_batched(x, y, a, b, 1.0, 1.0, 2.0, iters, "linesearch")
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            P.fw_solve_batched(x, y, a, b, 1.0, 1.0, 2.0, iters, "linesearch")
            e1.record(); torch.cuda.synchronize()
            out.append(e0.elapsed_time(e1))
        print(f"n=m={n} B={B}: {(out[1]-out[0])/50*1e3:.1f} us/iter")
