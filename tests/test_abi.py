"""The C-ABI library loads and exports every symbol include/uot_b200.h
declares (CPU-only: no compute calls)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_2201_00730_b200 import _lib


def header_symbols():
    text = open(os.path.join(ROOT, "include", "uot_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+char\s*\*|int)\s+(uot_\w+)\s*\(", text, re.M)))


def test_header_and_binding_agree():
    assert header_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_symbol():
    if not os.path.exists(_lib.SO_PATH):
        pytest.skip("extension not built")
    lib = ctypes.CDLL(_lib.SO_PATH)
    for name in header_symbols():
        assert hasattr(lib, name), name
    lib.uot_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.uot_version()


def test_descriptor_layouts():
    # field offsets of the ctypes mirrors follow the C struct order
    assert _lib.SinkhornDesc.shard_rows.offset > _lib.SinkhornDesc.nccl_comm.offset
    assert _lib.FwDesc.status.offset > _lib.FwDesc.summary.offset


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2201_00730_b200 as P

    a = P.DiscreteMeasure([0.0, 1.0], [0.5, 0.5])
    prob = P.UotProblem(a, a, P.PowerDistance(2.0), P.KL(1.0), P.KL(1.0), eps=0.1)
    with pytest.raises(P.UotError):
        P.h_sinkhorn_step(prob, P.DualPair.zeros(2, 2))


def test_product_never_imports_the_oracle():
    """oracle/ is the checker: nothing in the product package may import,
    link or execute it (there is no CPU fallback)."""
    import re

    pkg = os.path.join(ROOT, "paper_2201_00730_b200")
    offenders = []
    for dirpath, _, files in os.walk(pkg):
        for name in files:
            if not name.endswith((".py", ".cu", ".cuh")):
                continue
            text = open(os.path.join(dirpath, name), encoding="utf-8").read()
            if re.search(r"^\s*(import oracle|from oracle|import\s+oracle\b)|_oracle\.so|oracle_smin",
                         text, re.M):
                offenders.append(name)
    assert offenders == []
