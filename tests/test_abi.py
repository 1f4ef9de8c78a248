"""The C-ABI library: builds, loads, exports every declared symbol, struct layouts agree with the
header, and argument errors map to the reference's exception classes — all without a GPU."""

import ctypes as C
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

from paper_2511_03126_b200 import _lib
from paper_2511_03126_b200.build import ROOT, build
from paper_2511_03126_b200.errors import BundleStructureError

HEADER = os.path.join(ROOT, "include", "propfield_b200.h")


@pytest.fixture(scope="module")
def lib():
    build()
    return _lib.load()


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w]+\*?\s+\*?(pf_\w+)\(", src, re.M)))


def test_header_declares_the_path(lib):
    syms = declared_symbols()
    for must in ("pf_visible_in_view", "pf_bilinear_gather", "pf_accumulate_features",
                 "pf_visibility_mask", "pf_aggregate_features", "pf_material_similarity",
                 "pf_softmax_weights", "pf_regress_with_weights", "pf_voxel_mass", "pf_fuse_query"):
        assert must in syms


def test_every_declared_symbol_is_exported_and_bound(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (pf_\w+)", out))
    for s in declared_symbols():
        assert s in exported, s
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature"


def test_struct_layouts_match_header(lib):
    """Compile a probe against the header with gcc and compare sizes/offsets with ctypes."""
    fields = [f for f, _ in _lib.FuseArgs._fields_]
    probe = "#include <stdio.h>\n#include <stddef.h>\n#include \"propfield_b200.h\"\nint main(){\n"
    probe += 'printf("%zu %zu\\n", sizeof(pf_view_t), sizeof(pf_fuse_args_t));\n'
    for f in fields:
        probe += f'printf("%zu\\n", offsetof(pf_fuse_args_t, {f}));\n'
    for f in _lib.VIEW_DTYPE.names:
        probe += f'printf("%zu\\n", offsetof(pf_view_t, {f}));\n'
    probe += "return 0;}\n"
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "p.c")
        exe = os.path.join(d, "p")
        open(c, "w").write(probe)
        subprocess.run(["gcc", "-I", os.path.dirname(HEADER), c, "-o", exe], check=True)
        vals = [int(x) for x in subprocess.run([exe], capture_output=True, text=True,
                                               check=True).stdout.split()]
    assert vals[0] == _lib.VIEW_DTYPE.itemsize == 160
    assert vals[1] == C.sizeof(_lib.FuseArgs)
    for f, off in zip(fields, vals[2 : 2 + len(fields)]):
        assert getattr(_lib.FuseArgs, f).offset == off, f
    for f, off in zip(_lib.VIEW_DTYPE.names, vals[2 + len(fields) :]):
        assert _lib.VIEW_DTYPE.fields[f][1] == off, f


def test_abi_version(lib):
    assert lib.pf_abi_version() == 1


def test_value_error_maps_without_touching_the_gpu(lib):
    # argument validation happens before any CUDA call (grounding.py:170-171 semantics)
    rc = lib.pf_softmax_weights(None, 4, 3, 0.0, None, None, None, None)
    assert rc == _lib.PF_ERR_VALUE
    with pytest.raises(ValueError, match="temperature must be positive"):
        _lib.check(rc)


def test_structure_error_maps(lib):
    rc = lib.pf_bilinear_gather(None, _lib.PF_F32, 0, 4, 4, None, None, 10, None, None)
    assert rc == _lib.PF_ERR_STRUCTURE
    with pytest.raises(BundleStructureError):
        _lib.check(rc)


def test_fuse_rejects_bad_shapes(lib):
    rec = np.zeros(1, dtype=_lib.VIEW_DTYPE)
    a = _lib.FuseArgs()
    a.n, a.nviews, a.views_host, a.views = 10, 1, rec.ctypes.data, 1
    a.d, a.k, a.p, a.temperature, a.grid = 2048, 4, 2, 0.1, 8
    assert lib.pf_fuse_query(C.byref(a), None) == _lib.PF_ERR_STRUCTURE
    a.d, a.temperature = 64, -1.0
    assert lib.pf_fuse_query(C.byref(a), None) == _lib.PF_ERR_VALUE
    assert "temperature" in lib.pf_last_error().decode()


def test_sm100a_code_in_library(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2511_03126_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f
