"""The C-ABI library loads without a GPU and exports every symbol include/bq.h declares."""
import ctypes
import re
from pathlib import Path

from paper_2307_02043_b200 import _abi

HEADER = Path(__file__).resolve().parent.parent / "include" / "bq.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bq_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _abi.load_library()
    names = declared_symbols()
    assert names, "no declarations parsed"
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(_abi.EXPORTS), (set(names) ^ set(_abi.EXPORTS))


def test_version_and_error_without_gpu():
    lib = _abi.load_library()
    assert lib.bq_version().startswith(b"bq ")
    assert isinstance(lib.bq_last_error(), bytes)


def test_struct_layout_matches_header(tmp_path):
    """ctypes mirrors of bq_wtv_desc / bq_wtv_report agree with the C compiler."""
    import shutil
    import subprocess

    import pytest

    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    src = tmp_path / "layout.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "bq.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu %zu\\n\", sizeof(bq_wtv_desc), sizeof(bq_wtv_report),"
        " offsetof(bq_wtv_desc, report), offsetof(bq_wtv_report, newton_residual), sizeof(bq_slab_desc),"
        " offsetof(bq_slab_desc, tau));return 0;}\n"
    )
    exe = tmp_path / "layout"
    subprocess.run([cc, "-I", str(HEADER.parent), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert got == [
        ctypes.sizeof(_abi.WtvDesc),
        ctypes.sizeof(_abi.WtvReport),
        _abi.WtvDesc.report.offset,
        _abi.WtvReport.newton_residual.offset,
        ctypes.sizeof(_abi.SlabDesc),
        _abi.SlabDesc.tau.offset,
    ]
