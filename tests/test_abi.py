"""The C-ABI library loads and exports every symbol include/bnfft.h declares (no GPU needed),
and its host-side validation rejects bad options before touching a device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bnfft.h")
LIB = os.path.join(ROOT, "paper_2502_07155_b200", "libbnfft.so")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"BNFFT_API\s+[\w\s\*]+?\b(bnfft_\w+)\s*\(", src)))


def test_header_declares_api():
    syms = declared_symbols()
    for s in ("bnfft_plan_create", "bnfft_set_nodes", "bnfft_execute", "bnfft_destroy",
              "bnfft_precompute", "bnfft_transform_host", "bnfft_get_info"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "run __graft_entry__.build()"
    lib = ctypes.CDLL(LIB)
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_binding_wraps_every_symbol():
    from paper_2502_07155_b200 import bnfft
    assert set(declared_symbols()) == set(bnfft.EXPORTED)
    assert b"sm_100a" in bnfft.bnfft_build_info()


def test_library_is_sm100a_cubin():
    """The kernels are compiled for sm_100a (no PTX JIT, no other arch)."""
    import subprocess
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", r.stdout))
    assert arches == {"100a"}, arches


@pytest.mark.parametrize("kw,code", [
    (dict(d=4), "BNFFT_E_BAD_DIM"),
    (dict(M=7), "BNFFT_E_BAD_BANDWIDTH"),
    (dict(M=0), "BNFFT_E_BAD_BANDWIDTH"),
    (dict(sigma=0.5), "BNFFT_E_BAD_SIGMA"),
    (dict(m=0), "BNFFT_E_TRUNCATION_TOO_LARGE"),
    (dict(M=8, m=8), "BNFFT_E_TRUNCATION_TOO_LARGE"),
    (dict(window=9), "BNFFT_E_BAD_WINDOW_PARAM"),
    (dict(d=3, m=9, M=64), "BNFFT_E_UNSUPPORTED"),
    (dict(sigma=1.0, window=1), "BNFFT_E_BAD_WINDOW_PARAM"),
    (dict(batch=0), "BNFFT_E_INVALID_ARG"),
])
def test_option_validation_without_device(kw, code):
    from paper_2502_07155_b200 import bnfft
    o = dict(d=1, M=64, sigma=2.0, m=5, window=0, shape=0.0, prec=1, batch=1, flags=0, device=0, stream=None)
    o.update(kw)
    h = ctypes.c_void_p()
    rc = bnfft.bnfft_plan_create(ctypes.byref(bnfft.bnfft_opts(**o)), ctypes.byref(h))
    assert bnfft.STATUS[rc] == code
    assert not h.value


def test_no_device_is_loud():
    """Valid options on a box without a CUDA device: BNFFT_E_CUDA, never a CPU fallback."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2502_07155_b200 import bnfft
    with pytest.raises(bnfft.BnfftError) as ei:
        bnfft.Plan(1, 64, 2.0, 5, stream=0)
    assert ei.value.code == bnfft.BNFFT_E_CUDA


def test_null_arguments():
    from paper_2502_07155_b200 import bnfft
    assert bnfft.bnfft_plan_create(None, None) == bnfft.BNFFT_E_INVALID_ARG
    assert bnfft.bnfft_set_nodes(None, 0, None, None) == bnfft.BNFFT_E_INVALID_ARG
    assert bnfft.bnfft_execute(None, None, None) == bnfft.BNFFT_E_INVALID_ARG
    assert bnfft.bnfft_destroy(None) == bnfft.BNFFT_OK
    assert bnfft.bnfft_status_string(-7) == b"node not finite"
