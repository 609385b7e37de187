"""CPU checks of the drop-in boundary: the product library loads and exports
every entry point include/fmoe_b200.h declares, and host-side error mapping
works without a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fmoe_b200.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int64_t|int)\s+(fmoe_\w+)\(", src, re.M)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("fmoe_gate_fwd", "fmoe_gate_bwd", "fmoe_plan_build", "fmoe_scatter", "fmoe_gather_combine",
                 "fmoe_scatter_bwd", "fmoe_gather_combine_bwd", "fmoe_experts_fwd", "fmoe_experts_bwd",
                 "fmoe_layer_fwd", "fmoe_layer_bwd", "fmoe_layer_step_host"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2103_13262_b200 import _lib

    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_lib.EXPORTS) >= set(declared())


def test_no_oracle_in_product_library():
    """The product must not link or embed the checkers."""
    from paper_2103_13262_b200 import _lib

    blob = open(_lib.LIB_PATH, "rb").read()
    for forbidden in (b"orc_", b"fmoe_ref", b"liborc", b"libfmoe_ref"):
        assert forbidden not in blob


def test_plan_sizes_and_shape_errors_on_host():
    import ctypes as C

    from paper_2103_13262_b200._lib import ShapeError, check, lib

    cap, scr = C.c_int64(), C.c_int64()
    check(lib.fmoe_plan_sizes(65536, 2, 64, 128, C.byref(cap), C.byref(scr)))
    assert cap.value % 128 == 0 and cap.value >= 131072 + 0
    assert cap.value <= 131072 + 64 * 128
    check(lib.fmoe_plan_sizes(3, 2, 3, 1, C.byref(cap), C.byref(scr)))
    assert cap.value == 6
    with pytest.raises(ShapeError):
        check(lib.fmoe_plan_sizes(3, 0, 3, 1, C.byref(cap), C.byref(scr)))
