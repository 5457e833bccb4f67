"""Host-side checks of the GF(2^256) extension (CPU): the modulus is the
first irreducible of the reference's scan order at q = 256 (_moduli.py:1-11,
restated in tools/gen_moduli.py), the field cap of the drop-in API is
unchanged, and the wide ABI rejects other widths without touching a GPU."""
import pathlib
import sys

import pytest

REPO = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO / "tools"))

import paper_2402_14607_b200 as bx  # noqa: E402
from paper_2402_14607_b200 import gf2q, wide  # noqa: E402
from paper_2402_14607_b200.errors import CapacityError  # noqa: E402


def test_wide_modulus_is_irreducible_and_first_in_scan():
    import gen_moduli

    assert gf2q.is_irreducible(wide.modulus_int(256))
    assert gen_moduli.first_modulus(256) == wide.WIDE_MODULI[256]


def test_drop_in_api_keeps_the_reference_cap():
    with pytest.raises(CapacityError):
        bx.field(129)
    with pytest.raises(CapacityError):
        wide.modulus_int(192)


def test_wide_abi_rejects_other_widths():
    from paper_2402_14607_b200 import _lib
    try:
        L = _lib.lib()
    except Exception:  # noqa: BLE001 - library not built here
        pytest.skip("library not built")
    assert L.bx_extract_eq_wide(None, 0, None, 0, 128, 4, 1, None, 0, None) == _lib.BX_ERANGE
    assert b"q = 256" in L.bx_last_error()
    assert L.bx_extract_eq_wide(None, 0, None, 0, 256, 4, 0, None, 0, None) == 0
