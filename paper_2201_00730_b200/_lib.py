"""ctypes binding of the C-ABI in include/uot_b200.h (``_uot_b200.so``).

The product path has no CPU fallback: if the shared library is missing, or no
CUDA device is present, every solver call raises.  Status codes are mapped
onto the reference's exception classes (src/exceptions.py:4-25).
"""

from __future__ import annotations

import ctypes
import os

from . import exceptions as E

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("UOT_B200_LIB") or os.path.join(_HERE, "_uot_b200.so")

UOT_OK = 0
F32, F64 = 0, 1
SINKHORN_F, SINKHORN_H, SINKHORN_G = 0, 1, 2
ENT_KL, ENT_BERG, ENT_BALANCED = 0, 1, 2
COST_SQEUCLID, COST_POWER, COST_EXPLICIT = 0, 1, 2
STEP_HARMONIC, STEP_LINESEARCH, STEP_PAIRWISE = 0, 1, 2

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_f64 = ctypes.c_double


class SinkhornDesc(ctypes.Structure):
    _fields_ = [
        ("variant", _i32), ("dtype", _i32), ("cost", _i32),
        ("batch", _i32), ("n", _i32), ("m", _i32), ("d", _i32),
        ("p", _f64), ("eps", _f64), ("rho1", _f64), ("rho2", _f64),
        ("x", _vp), ("y", _vp), ("c", _vp), ("ct", _vp), ("a", _vp), ("b", _vp),
        ("f", _vp), ("g", _vp),
        ("init_given", _i32), ("iters", _i32), ("tol", _f64), ("use_tol", _i32),
        ("trace_delta", _vp), ("iterations", _vp),
        ("nccl_comm", _vp), ("nranks", _i32), ("rank", _i32), ("shard_rows", _vp),
        ("ent1", _i32), ("ent2", _i32), ("lam_given", _i32), ("lam0", _f64),
        ("status", _vp), ("warm_shifts", _i32),
    ]


class FwDesc(ctypes.Structure):
    _fields_ = [
        ("batch", _i32), ("n", _i32), ("m", _i32),
        ("p", _f64), ("rho1", _f64), ("rho2", _f64),
        ("step", _i32), ("max_iters", _i32), ("gap_tol", _f64), ("early_exit", _i32),
        ("x", _vp), ("y", _vp), ("a", _vp), ("b", _vp), ("f", _vp), ("g", _vp),
        ("h0", _vp), ("fw_gap", _vp), ("pd_gap", _vp), ("iterations", _vp),
        ("ei", _vp), ("ej", _vp), ("em", _vp), ("count", _vp), ("summary", _vp),
        ("status", _vp), ("step_size", _vp), ("natoms", _vp), ("ref_f", _vp), ("err_f", _vp), ("c", _vp),
        ("ent1", _i32), ("ent2", _i32),
        ("step_in", _vp), ("away_in", _vp), ("supp_hash", _vp), ("supp_nnz", _vp),
    ]


class BaryDesc(ctypes.Structure):
    _fields_ = [
        ("batch", _i32), ("k", _i32), ("n", _i32),
        ("omega", _vp), ("lens", _vp), ("rho", _f64),
        ("step", _i32), ("max_iters", _i32), ("gap_tol", _f64), ("early_exit", _i32),
        ("x", _vp), ("a", _vp), ("f", _vp),
        ("h0", _vp), ("fw_gap", _vp), ("pd_gap", _vp), ("iterations", _vp),
        ("idx", _vp), ("mass", _vp), ("count", _vp), ("summary", _vp), ("status", _vp),
        ("step_in", _vp), ("supp_hash", _vp), ("supp_nnz", _vp),
    ]


# Every symbol include/uot_b200.h declares (tests check the .so exports them).
EXPORTS = (
    "uot_version", "uot_last_error", "uot_device_arch",
    "uot_sinkhorn_workspace_size", "uot_sinkhorn_run", "uot_sinkhorn_verify", "uot_kl_scalars",
    "uot_anderson_workspace_size", "uot_anderson_reset", "uot_anderson_step", "uot_anderson_weights",
    "uot_cost_matrix", "uot_cost_quadruple_diameter", "uot_updated_marginals", "uot_eval_primal",
    "uot_logdotexp", "uot_entropy_map", "uot_divergence",
    "uot_ot1d_workspace_size", "uot_ot1d_batched", "uot_fw1d_workspace_size", "uot_fw1d_run", "uot_feasibility_1d",
    "uot_feasibility_explicit", "uot_translation",
    "uot_mot1d_workspace_size", "uot_mot1d_batched", "uot_mot_certify", "uot_bary_workspace_size", "uot_bary_run",
    "uot_mot1d_states", "uot_mot1d_cost_duals", "uot_mot_certify_costs",
    "uot_nccl_unique_id", "uot_nccl_comm_init", "uot_nccl_comm_destroy",
)

_LIB = None


def load(require_gpu=True):
    """Load the shared library (and, by default, insist on a CUDA device)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(SO_PATH):
            raise E.UotError(
                f"CUDA extension not built ({SO_PATH} missing); run "
                "`python -m paper_2201_00730_b200.build` -- there is no CPU fallback")
        lib = ctypes.CDLL(SO_PATH)
        lib.uot_version.restype = ctypes.c_char_p
        lib.uot_last_error.restype = ctypes.c_char_p
        _i64 = ctypes.c_int64
        lib.uot_anderson_workspace_size.argtypes = [_i32, _i64, _i32, _vp]
        lib.uot_anderson_reset.argtypes = [_i32, _i64, _i32, _vp, ctypes.c_size_t, _vp]
        lib.uot_anderson_step.argtypes = [_i32, _i64, _i64, _i32, _f64, _vp, _vp, _vp, _vp, _vp,
                                          _vp, ctypes.c_size_t, _vp]
        lib.uot_anderson_weights.argtypes = [_i32, _i32, _vp, _f64, _vp, _vp, _vp]
        lib.uot_cost_matrix.argtypes = [_i32, _i32, _vp, _vp, _f64, _vp, _vp]
        lib.uot_translation.argtypes = [_i32, _i32, _i32, _vp, _vp, _vp, _vp, _i32, _i32, _f64,
                                        _f64, _i32, _f64, _f64, _i32, _vp, _vp, _vp, _vp, _vp,
                                        _vp]
        lib.uot_feasibility_explicit.argtypes = [_i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp]
        lib.uot_cost_quadruple_diameter.argtypes = [_i32, _i32, _vp, _vp, _vp]
        lib.uot_updated_marginals.argtypes = [_i32, _i32, _vp, _vp, _vp, _vp, _f64, _f64, _f64,
                                              _vp, _vp, _vp]
        lib.uot_logdotexp.argtypes = [_i64, _i64, _i64, _vp, _vp, _f64, _vp, _vp]
        lib.uot_entropy_map.argtypes = [_i32, _i32, _f64, _f64, _i64, _vp, _vp, _vp, _vp]
        lib.uot_divergence.argtypes = [_i32, _f64, _i64, _vp, _vp, _vp, _vp]
        lib.uot_eval_primal.argtypes = [_i32, _i32, _vp, _vp, _f64, _vp, _vp, _vp, _i32, _vp, _vp,
                                        _vp, _i32, _i32, _f64, _f64, _f64, _vp, _vp]
        _LIB = lib
    if require_gpu:
        import torch

        if not torch.cuda.is_available():
            raise E.UotError("no CUDA device: the B200 kernels cannot run (no CPU fallback)")
    return _LIB


def check(status, what=""):
    if status == UOT_OK:
        return
    msg = (_LIB.uot_last_error() or b"").decode() if _LIB is not None else ""
    msg = f"{what}: {msg}" if what else msg
    if status == 1:
        raise E.MassBalanceError(msg)
    if status == 2:
        raise E.UnsupportedEntropyError(msg)
    if status == 3:
        raise ValueError(msg)
    if status == 6:
        raise E.InfeasibleDualError(msg)
    raise E.UotError(f"device failure ({status}): {msg}")


def ptr(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def stream_handle(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)
