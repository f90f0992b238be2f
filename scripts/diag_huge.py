import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import oracle as O
import paper_2201_00730_b200 as P
from paper_2201_00730_b200 import _device as D
from paper_2201_00730_b200 import synthetic as S
for n, m in [(3000, 2800), (16000, 15000), (20000, 18000), (30000, 20000)]:
    a, _ = S.mixture_measure(n, 5)
    b, _ = S.mixture_measure(m, 6)
    r = P.fw_solve_batched(a.points, b.points, a.weights, b.weights, 0.5, 0.5, 2.0, 6, "harmonic")
    out = O.fw_fixed(a.points, b.points, a.weights, b.weights, 0.5, 0.5, 6, step="harmonic")
    f, g = D.to_np(r.f[0]), D.to_np(r.g[0])
    df, dg = f - out["f"], g - out["g"]
    print(n, m, "h0 err", np.abs(D.to_np(r.h0[0]) - out["h0"]).max(),
          "df mean/ptp", df.mean(), np.ptp(df), "dg mean/ptp", dg.mean(), np.ptp(dg), flush=True)
