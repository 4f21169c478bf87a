"""The shared-reciprocal division used by strict mode equals __ddiv_rn bitwise."""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cuda", "_bin", "libdivcheck.so")


@pytest.mark.parametrize("regime", [0, 1, 2, 3])
def test_shared_reciprocal_division_is_ddiv_rn(regime):
    if not os.path.exists(LIB):
        pytest.fail(f"{LIB} not built (make -C tests/cuda)")
    lib = C.CDLL(LIB)
    lib.divcheck.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p]
    bad = C.c_ulonglong(0)
    ex = np.zeros(4)
    n = 1 << 28
    assert lib.divcheck(n, 0x1234 + regime, regime, C.byref(bad), ex.ctypes.data) == 0
    assert bad.value == 0, f"{bad.value} mismatches; e.g. a={ex[0]!r} b={ex[1]!r} got={ex[2]!r} want={ex[3]!r}"
