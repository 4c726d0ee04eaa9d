"""CPU checks of the C-ABI library: it loads, exports every symbol include/ieti.h declares,
and reports errors as return codes (no GPU needed)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ieti.h")).read()
    return sorted(set(re.findall(r"\b(ieti_[a-z_]+)\s*\(", src)))


def test_header_and_library_exports():
    import paper_1705_04531_b200 as lib
    syms = declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib._lib, s), s
    assert set(lib.EXPORTS) == set(syms)


def test_setup_without_gpu_is_an_error_code():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1705_04531_b200 as lib
    from workloads import make_workload
    with pytest.raises(lib.IetiError) as e:
        lib.Ieti.from_workload(make_workload("C1"))
    assert e.value.code in (-6, -8)


def test_null_args():
    import paper_1705_04531_b200 as lib
    h = ctypes.c_void_p()
    assert lib._lib.ieti_setup(None, ctypes.byref(h)) == -1
    assert lib._lib.ieti_last_error(None)
