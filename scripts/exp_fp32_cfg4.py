"""Experiment: fp32 error growth on cfg4_small (d=64) vs fp64 trajectory."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2201_00730_b200 as P
from paper_2201_00730_b200 import _device as D
from conftest import golden

z = golden("cfg4_small.npz")
x, y, a, b = z["x"][None], z["y"][None], z["alpha"][None], z["beta"][None]
eps, rho = float(z["eps"]), float(z["rho"])
C = ((z["x"][:, None, :] - z["y"][None, :, :]) ** 2).sum(-1)
for variant in ("h", "f"):
    for T in (1, 5, 20, 100, 300):
        f64, g64, _, _ = P.sinkhorn_batched(x, y, a, b, eps, rho, rho, T, variant=variant, precision="fp64")
        f64 = D.to_np(f64)[0]; g64 = D.to_np(g64)[0]
        out = [variant, T]
        for cost, kw in (("sqeuclid", {}), ("explicit", {"c": C[None]})):
            f32, g32, _, _ = P.sinkhorn_batched(x, y, a, b, eps, rho, rho, T, variant=variant, cost=cost,
                                                precision="fp32", **kw)
            df = D.to_np(f32)[0].astype(float) - f64
            dg = D.to_np(g32)[0].astype(float) - g64
            out += [cost, f"max {max(abs(df).max(), abs(dg).max()):.2e}", f"meanf {df.mean():.2e}",
                    f"meang {dg.mean():.2e}", f"resid {max(abs(df-df.mean()).max(), abs(dg-dg.mean()).max()):.2e}"]
        print(*out, flush=True)
