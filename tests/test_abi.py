"""CPU-side checks of the boundary: libfmm.so builds for sm_100a, loads, exports every
symbol include/fmm.h declares, and refuses to run without a device (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    from paper_1405_7487_b200 import build
    return build.build()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "fmm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fmm_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(libpath):
    names = header_symbols()
    assert len(names) >= 15
    lib = C.CDLL(libpath)
    for n in names:
        assert hasattr(lib, n), n
    from paper_1405_7487_b200.fmm import SYMBOLS
    assert sorted(SYMBOLS) == names


def test_sm100a_only(libpath):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    assert not re.search(r"sm_(?!100a)\d+", out.stdout)


def test_no_oracle_in_product():
    # the product path never imports, links or includes the oracle
    pkg = os.path.join(ROOT, "paper_1405_7487_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "fmm_oracle" not in txt and "ofmm_" not in txt, f


def test_version_and_no_device(libpath):
    import torch
    from paper_1405_7487_b200 import FMM, FMMError, lib
    assert lib().fmm_version() >= 1
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(FMMError):
        FMM(100, 4, 0.5, 8, "f64")


def test_bad_arguments_rejected_before_device(libpath):
    from paper_1405_7487_b200 import lib
    h = C.c_void_p()
    for args in [(-1, 4, 0.5, 8, 1), (10, 0, 0.5, 8, 1), (10, 17, 0.5, 8, 1), (10, 4, 1.0, 8, 1),
                 (10, 4, 0.0, 8, 1), (10, 4, 0.5, 0, 1), (10, 4, 0.5, 8, 7)]:
        assert lib().fmm_create(*args, 0, C.byref(h)) == 1   # FMM_ERR_ARG
