"""The C-ABI boundary: every symbol declared in include/*.h is exported by the
in-tree libraries, the ctypes mirror declares exactly those symbols, and the
product fails loudly (no CPU fallback) when no GPU is present."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_1402_4247_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(kbg_\w+)\s*\(", src, flags=re.M)))


def exported(so):
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


@pytest.mark.parametrize("header,so,mirror", [
    ("kbgrid.h", _abi.KBGRID_SO, _abi.KBGRID_SYMBOLS),
    ("kbgsynth.h", _abi.KBGSYNTH_SO, _abi.KBGSYNTH_SYMBOLS),
])
def test_header_symbols_exported(built, header, so, mirror):
    names = declared(header)
    assert names, header
    ex = exported(so)
    missing = [n for n in names if n not in ex]
    assert not missing, f"{so} does not export {missing}"
    assert sorted(n for n, _, _ in mirror) == names


def test_library_loads_and_binds(built):
    lib = _abi.kbgrid()
    assert lib.kbg_version().decode().startswith("kbgrid")
    assert lib.kbg_status_string(_abi.KBG_ERR_CONSISTENCY) == b"consistency error"


def test_kernels_are_sm100a(built):
    out = subprocess.run(["cuobjdump", "-lelf", _abi.KBGRID_SO], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _abi.KBGRID_SO], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass  # FP64 tensor-core path of the grid kernels


def test_no_cpu_fallback_without_gpu(built):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1402_4247_b200.errors import CudaError
    from paper_1402_4247_b200.grid import GridPass
    from paper_1402_4247_b200.system import Fe3O4

    f = Fe3O4.config("primitive14_150Ry")
    with pytest.raises(CudaError):
        GridPass(f.system)


def test_null_arguments_are_config_errors(built):
    lib = _abi.kbgrid()
    h = C.c_void_p()
    assert lib.kbg_create(None, 0, C.byref(h)) == _abi.KBG_ERR_CONFIG
    assert lib.kbg_build_index(None) == _abi.KBG_ERR_CONFIG
    assert lib.kbg_density(None, 1, None, None) == _abi.KBG_ERR_CONFIG


def test_header_constants_match_python_mirror():
    """Every #define KBG_* integer constant of include/kbgrid.h has the same value in _abi.py (options,
    status codes): the Python mirror cannot drift from the C-ABI."""
    import os
    import re

    from paper_1402_4247_b200 import _abi

    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "kbgrid.h")).read()
    consts = dict(re.findall(r"^#define (KBG_[A-Z0-9_]+) (-?\d+)\b", hdr, flags=re.M))
    assert "KBG_OPT_EXCHANGE_SMS" in consts
    missing = [k for k in consts if not hasattr(_abi, k)]
    wrong = [k for k, v in consts.items() if hasattr(_abi, k) and getattr(_abi, k) != int(v)]
    assert not wrong, wrong
    # options must all be mirrored; other constants (sizes, status codes) where the mirror has them
    assert not [k for k in missing if k.startswith("KBG_OPT_")], missing
