"""The C-ABI library loads and exports every symbol include/saga.h declares
(CPU-only: no compute call is made without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "saga.h")


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2009_00804_b200 as saga
    return saga


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(saga_[a-z_]+)\s*\(", txt)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("saga_graph_build", "saga_layer", "saga_free"):     # BASELINE.json north_star
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (saga_[a-z_]+)\b", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    assert sorted(lib.EXPORTS) == declared_functions()
    # nothing else leaks out of the library (hidden visibility)
    extra = [n for n in re.findall(r"\bT (\S+)", out) if not n.startswith("saga_") and not n.startswith("_")]
    assert len(extra) < 50


def test_abi_version_and_error_string(lib):
    assert lib.saga_abi_version() == 4
    assert isinstance(lib.saga_last_error(), str)


def test_struct_layouts_match_header(lib, tmp_path):
    """ctypes mirrors vs the C compiler's view of include/saga.h (size and
    every field offset), so a header change cannot drift from the binding."""
    fields = {"saga_tensor": lib.saga_tensor, "saga_layer_opts": lib.saga_layer_opts,
              "saga_weights": lib.saga_weights}
    lines = []
    for name, cls in fields.items():
        lines.append(f'printf("%zu\\n", sizeof({name}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("%zu\\n", offsetof({name}, {fname}));')
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "saga.h"\nint main(void) {\n'
                   + "\n".join(lines) + "\nreturn 0;\n}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()]
    want = []
    for cls in fields.values():
        want.append(ctypes.sizeof(cls))
        want.extend(getattr(cls, f).offset for f, _ in cls._fields_)
    assert got == want


def test_product_package_has_no_oracle_or_fallback():
    """The product path never imports the oracle nor a CPU path."""
    pkg = os.path.join(ROOT, "paper_2009_00804_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "oracle.h" not in src, f
