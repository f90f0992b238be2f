"""tcgen05 kind::tf32 issue-rate probe (cycles per 128 x N x 8 MMA)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2201_00730_b200 import _lib
lib = _lib.load()
for ctas in (148,):
    for n in (64, 128, 256):
        for ss in (0, 1, 2, 3):
            if (ss == 2 and n > 128) or (ss == 3 and n > 64):
                continue
            out = torch.zeros(1, dtype=torch.int64, device="cuda")
            reps = 2000
            rc = lib.uot_probe_tc_rate(ctas, reps, n, ss, ctypes.c_void_p(out.data_ptr()), None)
            torch.cuda.synchronize()
            cyc = out.item() / ctas / reps
            print(f"ctas={ctas:3d} N={n:3d} {['ts','ss','ts-2acc','ts-4acc'][ss]}: {cyc:7.1f} cycles/MMA "
                  f"(floor 128*N/256 = {128 * n / 256:.0f})", flush=True)
