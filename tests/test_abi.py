"""The C-ABI library loads and exports every symbol include/stencil.h declares.

CPU-only (no compute calls): symbol table, version string, argument
validation paths that return before touching a device, and the host-only
slab planner.
"""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2301_11389_b200 import build, binding
    build.build()
    return binding.lib()


def header_functions():
    src = open(os.path.join(ROOT, "include", "stencil.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(stencil_[a-z_0-9]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(L):
    from paper_2301_11389_b200 import binding
    names = header_functions()
    assert len(names) >= 14
    assert sorted(binding.EXPORTS) == names
    for n in names:
        assert hasattr(L, n), n


def test_exports_are_c_linkage():
    out = os.popen(f"nm -D --defined-only {ROOT}/paper_2301_11389_b200/libstencil_b200.so").read()
    for n in header_functions():
        assert re.search(rf"\bT {n}\b", out), n


def test_library_is_built_for_sm_100a():
    out = os.popen(f"cuobjdump -lelf {ROOT}/paper_2301_11389_b200/libstencil_b200.so").read()
    assert "sm_100a" in out


def test_version(L):
    assert b"sm_100a" in L.stencil_version()


def _create(L, kind, dims, dtype, coeffs=None):
    h = ctypes.c_void_p()
    d = (ctypes.c_int64 * len(dims))(*dims)
    cp = (ctypes.c_double * len(coeffs))(*coeffs) if coeffs else None
    rc = L.stencil_create(ctypes.byref(h), kind, len(dims), d, dtype, cp, len(coeffs or []))
    return rc, h


def test_create_validation_errors(L):
    from paper_2301_11389_b200.binding import KINDS, DTYPES
    assert _create(L, 99, (8, 8), 1)[0] == -1                                   # unknown kind
    assert _create(L, KINDS["gameoflife"], (8, 8), DTYPES["f32"])[0] == -2      # GoL is int only
    assert _create(L, KINDS["jacobi2d5"], (8, 8), DTYPES["i32"])[0] == -2
    assert _create(L, KINDS["jacobi2d5"], (8, 8, 8), DTYPES["f32"])[0] == -1    # wrong ndims
    assert _create(L, KINDS["gaussblur5x5"], (8, 4), DTYPES["f32"])[0] == -1    # 4 < lo+hi+1
    assert _create(L, KINDS["jacobi2d5"], (10, 8), DTYPES["f32"])[0] == -3      # 40 B rows
    assert _create(L, KINDS["jacobi2d5"], (8, 8), DTYPES["f32"], [1.0])[0] == -1  # ncoeffs
    assert L.stencil_last_error()


def test_slab_plan_is_exported_host_logic(L):
    from paper_2301_11389_b200 import binding
    p = binding.slab_plan(16, 1, 1, 0, 2)
    assert p["own_end"] - p["own_begin"] == 8


def _header_enum(name):
    """{enumerator: value} of `enum <name> { ... };` in include/stencil.h."""
    src = open(os.path.join(ROOT, "include", "stencil.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    body = re.search(r"enum\s+" + name + r"\s*\{(.*?)\};", src, flags=re.S).group(1)
    out, nxt = {}, 0
    for item in (t.strip() for t in body.split(",")):
        if not item:
            continue
        k, _, v = item.partition("=")
        nxt = int(v.strip(), 0) if v.strip() else nxt
        out[k.strip()] = nxt
        nxt += 1
    return out


def test_binding_constants_match_the_header():
    """The binding's name -> value maps are the header's enums (kinds,
    dtypes, variants incl. ST_AUTO): argument marshalling only, no drift."""
    from paper_2301_11389_b200 import binding
    kinds = _header_enum("stencil_kind")
    assert {("ST_" + k.upper()): v for k, v in binding.KINDS.items()} == kinds
    dtypes = _header_enum("stencil_dtype")
    assert {("ST_" + k.upper()): v for k, v in binding.DTYPES.items()} == dtypes
    variants = _header_enum("stencil_variant")
    assert {("ST_" + k.upper()): v for k, v in binding.VARIANTS.items()} == variants
    assert variants["ST_AUTO"] == binding.VARIANTS["auto"]
