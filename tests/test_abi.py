"""CPU checks of the C-ABI boundary (-m "not gpu"): the library builds for sm_100a, loads,
and exports every symbol include/andes.h declares; the SASS contains the bulk-copy (TMA)
path of the timeline scan.  No compute calls (no GPU here)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2404_16283_b200 import build
    return build.build()


def _declared():
    src = open(os.path.join(ROOT, "include", "andes.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(andes_\w+)\s*\(", src, re.M)))


def test_header_declares_the_boundary():
    names = _declared()
    for need in ["andes_create", "andes_destroy", "andes_last_error", "andes_qoe_eval",
                 "andes_gain_estimate", "andes_schedule", "andes_schedule_host", "andes_version"]:
        assert need in names


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (andes_\w+)", out))
    assert set(_declared()) <= exported, set(_declared()) - exported


def test_binding_loads_and_matches_exports(libpath):
    import paper_2404_16283_b200 as A
    L = A.lib()
    for name in A.EXPORTS:
        assert hasattr(L, name)
    assert A.version().startswith("andes-b200")


def test_sm100a_cubin_and_bulk_copy(libpath):
    sass = subprocess.run(["cuobjdump", "-sass", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", libpath], capture_output=True, text=True).stdout
    assert "UTMALDG" in sass  # cp.async.bulk.tensor: TMA tile loads of the timeline scan
    assert "SYNCS" in sass    # mbarrier transaction completion


def test_no_gpu_raises_loudly(libpath):
    import torch
    import paper_2404_16283_b200 as A
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(A.AndesError):
        A.Context(16)
