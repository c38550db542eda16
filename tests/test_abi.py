"""The C-ABI library loads and exports every symbol include/dit.h declares (no GPU needed)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "dit.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\**\s*(di_[a-z_]+)\s*\(", src, flags=re.M)))


def test_library_exports_header_symbols():
    from paper_1501_06350_b200 import build
    lib_path = build.build()
    lib = ctypes.CDLL(lib_path)
    names = _declared()
    assert len(names) >= 11, names
    for name in names:
        assert hasattr(lib, name), f"{name} declared in include/dit.h but not exported"


def test_binding_names_match_header():
    from paper_1501_06350_b200 import build
    build.build()
    from paper_1501_06350_b200 import _lib
    assert sorted(_lib.EXPORTS) == _declared()
    for name in _declared():
        assert callable(getattr(_lib, name))


def test_opts_defaults_without_gpu():
    from paper_1501_06350_b200 import build
    build.build()
    from paper_1501_06350_b200 import _lib
    o = _lib.di_solve_opts_default()
    assert o.theta == 1.0 and o.variant == _lib.DI_VARIANT_AUTO and o.max_sweeps > 0
    assert _lib.di_last_error() == ""
