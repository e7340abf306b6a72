"""CPU checks of the product artefact: the C-ABI library loads, exports every
symbol include/nqb.h declares, fails loudly without a B200, and its host-only
entry points (status kinds, the rank rule) match the reference."""
import ctypes as C
import os
import re
import shutil
import subprocess

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "nqb.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nqb_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree(nq):
    assert declared_functions() == nq._lib.exported_symbols()


def test_library_exports_every_declared_symbol(nq):
    lib = nq._lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    if shutil.which("nm"):
        out = subprocess.run(["nm", "-D", "--defined-only", nq._lib.LIB_PATH],
                             capture_output=True, text=True, check=True).stdout
        exported = set(re.findall(r" T (nqb_\w+)", out))
        assert set(declared_functions()) <= exported


def test_no_cpu_path_without_device(nq):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib = nq._lib.load()
    h = C.c_void_p()
    assert lib.nqb_create(0, C.byref(h)) == 66  # NQB_E_NO_DEVICE
    assert b"no CPU path" in lib.nqb_last_error()
    with pytest.raises(nq.DeviceError):
        nq.Context(0)


def test_status_kinds(nq):
    lib = nq._lib.load()
    assert [lib.nqb_status_kind(c) for c in (0, 1, 4, 9, 11, 32, 33, 64, 66)] == \
        [0, 1, 1, 1, 1, 2, 2, 3, 3]
    assert nq.ZeroMatrix.kind == "numerical" and nq.CorruptPadding.kind == "validation"


def test_rank_rule_matches_reference(nq, chk):
    rng = chk.rng(94)
    for _ in range(300):
        n, m = 1 + int(rng.index(20000)), 1 + int(rng.index(20000))
        t = float(rng.uniform(0.01, 4.0, 1)[0])
        try:
            want = chk.rank_for_target_bpw(n, m, t)
        except Exception as e:  # noqa: BLE001
            with pytest.raises(nq.TargetTooSmall):
                nq.rank_for_target_bpw(n, m, t)
            assert e.code == 8
            continue
        assert nq.rank_for_target_bpw(n, m, t) == want
    with pytest.raises(nq.TargetTooSmall):
        nq.rank_for_target_bpw(4096, 4096, 1e-4)
    assert nq.rank_for_target_bpw(2000, 2000, 0.01) == 1


def _sass():
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    from paper_2602_06694_b200 import _lib
    return subprocess.run([exe, "-sass", _lib.LIB_PATH], capture_output=True, text=True,
                          check=True).stdout


def test_sass_is_sm100a_with_fp64_tensor_cores():
    sass = _sass()
    assert "sm_100a" in sass
    assert "DMMA" in sass  # fp64 tensor-core GEMM of the ADMM (dgemm.cu)
