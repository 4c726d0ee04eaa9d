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


def test_setup_args_layout_matches_header(tmp_path):
    """The binding's ctypes mirror of ieti_setup_args has the C layout of include/ieti.h (size and
    every field offset, compiled here with gcc)."""
    import shutil
    import subprocess
    import paper_1705_04531_b200 as lib
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    fields = [f for f, _ in lib.SetupArgs._fields_]
    src = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{ROOT}/include/ieti.h"', "int main(void) {",
           '  printf("size %zu\\n", sizeof(ieti_setup_args));']
    src += [f'  printf("{f} %zu\\n", offsetof(ieti_setup_args, {f}));' for f in fields]
    src += ["  return 0;", "}"]
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-o", str(exe), str(c)])
    got = dict(line.split() for line in subprocess.check_output([str(exe)]).decode().splitlines())
    assert int(got["size"]) == ctypes.sizeof(lib.SetupArgs)
    for f in fields:
        assert int(got[f]) == getattr(lib.SetupArgs, f).offset, f
