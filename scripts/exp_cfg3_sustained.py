"""cfg3 as whole 200-iteration solves (the BASELINE config) back to back: iter/s and SM
clocks under the sustained load -- decides what bench.py's step should be."""
import os, sys, time, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2201_00730_b200 as P
from paper_2201_00730_b200 import synthetic as S
dev = torch.device("cuda:0")
c = S.cfg3_inputs()
x, y, a, b = (torch.as_tensor(v, dtype=torch.float32, device=dev) for v in (c.x, c.y, c.alpha, c.beta))
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
def solve():
    return P.sinkhorn_batched(x, y, a, b, c.eps, c.rho, c.rho, iters, variant="h", precision="fp32")
solve(); torch.cuda.synchronize()
for r in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); solve(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    q = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu,clocks_event_reasons.active", "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    print(f"rep {r}: {ms:.1f} ms  {iters / ms * 1e3:.1f} iter/s   [{q}]")
