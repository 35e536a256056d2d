"""C-ABI library checks that need no GPU: it loads, exports every symbol
include/gi.h declares, and rejects bad arguments without touching a device."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "gi.h")).read()
    return sorted(set(re.findall(r"^GI_API [\w\* ]+?\b(gi_\w+)\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def gi():
    from paper_1805_00923_b200 import build

    build.build()
    from paper_1805_00923_b200 import gi as _gi

    return _gi


def test_header_declares_boundary():
    names = _declared()
    for must in ("gi_graph_create", "gi_pagerank", "gi_bfs", "gi_context_create", "gi_last_error"):
        assert must in names
    assert len(names) >= 19


def test_library_exports_every_declared_symbol(gi):
    out = subprocess.run(["nm", "-D", "--defined-only", gi.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (gi_\w+)$", out, flags=re.M))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    # and nothing beyond the ABI leaks out of the .so
    assert exported == set(_declared())
    # the binding covers the same names
    assert set(gi.EXPORTED) == set(_declared())


def test_library_is_sm100a(gi):
    out = subprocess.run(["cuobjdump", "--list-elf", gi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_version(gi):
    assert gi.gi_abi_version() == 3
    for s, name in [(0, "GI_OK"), (1, "GI_ERR_INVALID_ARGUMENT"), (2, "GI_ERR_VERTEX_OUT_OF_RANGE"),
                    (4, "GI_ERR_CUDA"), (7, "GI_ERR_INTERNAL")]:
        assert gi._lib.gi_status_string(s).decode() == name


def test_argument_validation_without_device(gi):
    import ctypes

    out = ctypes.c_void_p()
    # NULL context
    st = gi._lib.gi_graph_create(None, 4, 0, None, None, 0, ctypes.byref(out))
    assert st == gi.GI_ERR_INVALID_ARGUMENT
    assert "NULL context" in gi._lib.gi_last_error().decode()
    # NULL graph handles
    assert gi._lib.gi_pagerank(None, 20, 0.85, None) == gi.GI_ERR_INVALID_ARGUMENT
    assert gi._lib.gi_bfs(None, 0, None) == gi.GI_ERR_INVALID_ARGUMENT
    assert gi._lib.gi_graph_destroy(None) == gi.GI_ERR_INVALID_ARGUMENT
    with pytest.raises(gi.GiError):
        gi.gi_graph_num_vertices(None)


def test_no_cpu_fallback(gi):
    """Without a CUDA device the library refuses (GI_ERR_CUDA) instead of computing on the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(gi.GiError) as e:
        gi.gi_context_create(0)
    assert e.value.status == gi.GI_ERR_CUDA


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1805_00923_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f), errors="replace").read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "gi_oracle" not in txt, f


def test_binding_constants_match_header(gi):
    """Every enum constant of include/gi.h the binding defines has the header's value."""
    src = open(os.path.join(ROOT, "include", "gi.h")).read()
    consts = {}
    for body in re.findall(r"enum\s*\{([^}]*)\}", src):
        for name, val in re.findall(r"\b(GI_[A-Z0-9_]+)\s*=\s*(-?\d+)\s*(?=,|/|$)", body.strip()):
            consts[name] = int(val)
    assert consts["GI_PR_PULL_PARTITIONED"] == 4
    checked = 0
    for name, val in consts.items():
        if hasattr(gi, name):
            assert getattr(gi, name) == val, name
            checked += 1
    assert checked >= 10
