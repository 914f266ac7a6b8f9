"""The device FPFH's frame-source decision (csrc/lk_acos_cr.hpp, used by
csrc/lk_prepare.cu swap_decision) assumes that this machine's libm acos --
the one the reference calls at proj/src/fpfh.cpp:28 -- returns the correctly
rounded value wherever the exact value is at least 0.05 ulp from a rounding
midpoint, and one of the midpoint's two neighbours otherwise. These check
the premise and the comparison built on it against the libm of the machine
the tests run on (the same image as the GPU box), through the same header
compiled into the fixture library."""
import ctypes as C
import math

import numpy as np

from paper_1801_01572_b200 import abi


def _sweep(fn, seed, n):
    d, w = C.c_int64(), C.c_int64()
    getattr(abi.synth_lib(), fn)(C.c_uint64(seed), C.c_int64(n), C.byref(d), C.byref(w))
    return d.value, w.value


def test_acos_cr_equals_libm_where_decided():
    decided, wrong = _sweep("lks_acos_cr_sweep", 12345, 4_000_000)
    assert wrong == 0
    assert decided > 0.85 * 4_000_000  # ~10 % lie within 0.05 ulp of a midpoint


def test_acos_greater_equals_libm_on_near_ties():
    # pairs a few ulps apart in either order, as on planar faces
    decided, wrong = _sweep("lks_acos_greater_sweep", 7, 4_000_000)
    assert wrong == 0
    assert decided > 0.9 * 4_000_000


def test_acos_order_beyond_threshold():
    # swap_decision settles |x1 - x2| > 2.5e-16 by the argument order alone
    checked, wrong = _sweep("lks_acos_threshold_sweep", 11, 4_000_000)
    assert wrong == 0 and checked > 3_900_000


def test_acos_cr_edge_arguments():
    L = abi.synth_lib()
    xs = np.array([0.0, 1.0, 0.5, math.cos(1.0), 1e-300, 5e-324, 0.999999, 0.9999999, 1.0 - 2.0 ** -53,
                   math.nextafter(0.0, 1.0), 0.7071067811865476, 0.8660254037844386, 1e-8, 0.25, 0.75])
    d, w = C.c_int64(), C.c_int64()
    L.lks_acos_cr_check(xs.ctypes.data_as(abi.dptr), C.c_int64(xs.size), C.byref(d), C.byref(w))
    # acos(0.5), acos(0.75) lie within 0.02 ulp of a midpoint and x within ~5e-7
    # of 1 is left to libm: those are undecided, never wrong
    assert w.value == 0 and d.value >= xs.size - 6
