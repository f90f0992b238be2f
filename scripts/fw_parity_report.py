"""Per-case FW parity report vs the reference goldens (GPU)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2201_00730_b200 as P
from paper_2201_00730_b200 import _device as D
from conftest import golden, cases, rel_err
z = golden("fw.npz")
for k in cases(z):
    r1, r2, p, iters, ls = z[f"c{k}_par"]
    step = "linesearch" if ls else "harmonic"
    r = P.fw_solve_batched(z[f"c{k}_x"], z[f"c{k}_y"], z[f"c{k}_a"], z[f"c{k}_b"], r1, r2, p, int(iters), step)
    h0 = D.to_np(r.h0[0]); ref = z[f"c{k}_h0"]
    rel = np.abs(h0 - ref) / np.abs(ref).max()
    bad = np.where(rel > 1e-9)[0]
    pe = rel_err(D.to_np(r.f[0]), D.to_np(r.g[0]), z[f"c{k}_f"], z[f"c{k}_g"])
    c = int(r.count[0].item())
    same = c == len(z[f"c{k}_i"]) and (D.to_np(r.ei[0, :c]) == z[f"c{k}_i"]).all() and (D.to_np(r.ej[0, :c]) == z[f"c{k}_j"]).all()
    print(f"case {k} {len(z[f'c{k}_x'])}x{len(z[f'c{k}_y'])} {step:10s} h0 max rel {rel.max():.2e} "
          f"bad iters {bad[:8].tolist()} ({len(bad)}) pot {pe:.2e} plan_same {same}", flush=True)
k = 7
r1, r2, p, iters, ls = z[f"c{k}_par"]
r = P.fw_solve_batched(z[f"c{k}_x"], z[f"c{k}_y"], z[f"c{k}_a"], z[f"c{k}_b"], r1, r2, p, 12, "linesearch")
print("case 7 gammas:", [f"{v:.15f}" for v in D.to_np(r.step_size[0])])
print("case 7 h0:", [f"{v:.17f}" for v in D.to_np(r.h0[0])])
