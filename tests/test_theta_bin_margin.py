"""The FP32 pre-check of the FPFH theta bin (csrc/lk_prepare.cu pair_bins):
tv = 11 (theta + pi) / 2 pi computed in float32 from float32 inputs stays
within 1e-5 of the FP64 value, so a float tv more than 1e-4 from every
integer decides the same bin as the reference's FP64 theta
(proj/src/fpfh.cpp:39-45). CPU check of the error budget with numpy's float32
arctan2 (CUDA's atan2f is within 3 ulp as well)."""
import numpy as np


def _tv32(y, x):
    tf = np.arctan2(y.astype(np.float32), x.astype(np.float32))
    return np.float32(11.0) * (tf + np.float32(3.14159265)) / np.float32(6.28318531)


def _tv64(y, x):
    return 11.0 * (np.arctan2(y, x) + np.pi) / (2.0 * np.pi)


def test_float_tv_within_budget():
    rng = np.random.default_rng(5)
    n = 2_000_000
    ang = rng.uniform(-np.pi, np.pi, n)
    # half the samples within 1e-3 rad of an inner bin edge
    k = rng.integers(1, 11, n // 2)
    ang[: n // 2] = -np.pi + 2 * np.pi * k / 11 + rng.uniform(-1e-3, 1e-3, n // 2)
    mag = 10.0 ** rng.uniform(-30, 30, n)
    y, x = np.sin(ang) * mag, np.cos(ang) * mag
    d = np.abs(_tv32(y, x).astype(np.float64) - _tv64(y, x))
    assert d.max() < 1e-5


def test_decided_bins_agree():
    rng = np.random.default_rng(6)
    ang = rng.uniform(-np.pi, np.pi, 1_000_000)
    y, x = np.sin(ang), np.cos(ang)
    tvf = _tv32(y, x)
    far = np.abs(tvf - np.rint(tvf)) > np.float32(1e-4)
    bf = np.clip(np.floor(tvf[far]).astype(int), 0, 10)
    b64 = np.clip(np.floor(_tv64(y[far], x[far])).astype(int), 0, 10)
    assert far.mean() > 0.99 and np.array_equal(bf, b64)
