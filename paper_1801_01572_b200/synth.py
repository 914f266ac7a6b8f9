"""Synthetic fixtures (host C++ generators in csrc/lk_synth.cpp).

Restatements of the reference's seeded generators (proj/src/synth.cpp) and
test helpers (proj/tests/support/helpers.hpp) plus the measurement configs of
SURVEY.md 8d. Input generation only -- never part of a timed region.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Tuple

import numpy as np

from . import abi
from .registration import PointCloud, RigidTransform


@dataclass
class RegistrationPair:
    """synth.hpp RegistrationPair: truth maps source points onto the target."""

    source: PointCloud
    target: PointCloud
    truth: RigidTransform
    overlap: float = 0.0


def _take(h, status) -> RegistrationPair:
    L = abi.synth_lib()
    if not h:
        msg = L.lks_last_error()
        raise RuntimeError(f"synth failed ({status.value}): {msg.decode() if msg else ''}")
    try:
        clouds = []
        for w in range(2):
            n = L.lks_count(h, w)
            if n < 0:
                clouds.append(None)
                continue
            xyz = np.empty((n, 3))
            nrm = np.empty((n, 3)) if L.lks_has_normals(h, w) else None
            L.lks_get(h, w, xyz.ctypes.data_as(abi.dptr), nrm.ctypes.data_as(abi.dptr) if nrm is not None else None)
            clouds.append(PointCloud(xyz, nrm))
        R, t, sc = np.empty(9), np.empty(3), C.c_double()
        if clouds[1] is not None:
            L.lks_truth(h, R.ctypes.data_as(abi.dptr), t.ctypes.data_as(abi.dptr), C.byref(sc))
            return RegistrationPair(clouds[0], clouds[1], RigidTransform(R.reshape(3, 3), t.copy()), sc.value)
        return RegistrationPair(clouds[0], None, RigidTransform(), 0.0)
    finally:
        L.lks_free(h)


def synth_registration_pair(seed: int, leaf: float = 0.05) -> RegistrationPair:
    """proj/src/synth.cpp:592-623"""
    st = C.c_int()
    return _take(abi.synth_lib().lks_registration_pair(seed, leaf, C.byref(st)), st)


def synth_negative_pair(seed: int, leaf: float = 0.05) -> RegistrationPair:
    """proj/src/synth.cpp:625-653"""
    st = C.c_int()
    return _take(abi.synth_lib().lks_negative_pair(seed, leaf, C.byref(st)), st)


def depth_frame_pair(seed: int = 1, boxes: int = 6, width: int = 640, height: int = 480, fx: float = 525.0,
                     fy: float = 525.0, cx: float = 319.5, cy: float = 239.5, stride: int = 1, noise: float = 0.005,
                     frames: int = 90, frame_a: int = 0, frame_b: int = 6) -> RegistrationPair:
    """Config B1/B2: two 640x480 renders of make_room_scene(1, 6)
    from the synth_scene orbit; truth maps frame_a's camera frame into frame_b's."""
    st = C.c_int()
    h = abi.synth_lib().lks_frame_pair(seed, boxes, width, height, fx, fy, cx, cy, stride, noise, frames, frame_a,
                                       frame_b, C.byref(st))
    return _take(h, st)


def submap_pair(seed: int = 2, boxes: int = 6, views: int = 8, width: int = 640, height: int = 480, stride: int = 1,
                noise: float = 0.005, frames: int = 90, a0: int = 0, b0: int = 8, step: int = 2) -> RegistrationPair:
    """Config D: world-frame unions of `views` renders of
    make_room_scene(seed) along two overlapping orbit arcs (~2.4M points each
    at 640x480, stride 1), no downsample; the source is displaced by
    random_transform(pi/3, 1 m) and truth maps it back onto the target."""
    st = C.c_int()
    h = abi.synth_lib().lks_submap_pair(seed, boxes, views, width, height, stride, noise, frames, a0, b0, step,
                                        C.byref(st))
    return _take(h, st)


def surface_pair(seed: int = 1, density: float = 1000.0, noise: float = 0.005) -> RegistrationPair:
    """Config A: Q = sample_surface(make_scatter_scene(seed)),
    P = T^-1 (Q + N(0, noise^2)); truth T = random_transform(RngStream(seed, 0xA110))."""
    st = C.c_int()
    return _take(abi.synth_lib().lks_surface_pair(seed, density, noise, C.byref(st)), st)


def random_cloud(n: int, seed: int, stream: int = 0, lo: float = -1.0, hi: float = 1.0,
                 with_normals: bool = False) -> PointCloud:
    """proj/tests/support/helpers.hpp:16-31 on RngStream(seed, stream)."""
    st = C.c_int()
    return _take(abi.synth_lib().lks_random_cloud(seed, stream, n, lo, hi, 1 if with_normals else 0, C.byref(st)),
                 st).source


def random_transform(seed: int, stream: int = 0, max_angle: float = math.pi * 0.9, max_trans: float = 1.0,
                     skip_draws: int = 0) -> RigidTransform:
    """proj/tests/support/helpers.hpp:34-46 on a fresh RngStream(seed, stream)."""
    R, t = np.empty(9), np.empty(3)
    abi.synth_lib().lks_random_transform(seed, stream, skip_draws, max_angle, max_trans,
                                         R.ctypes.data_as(abi.dptr), t.ctypes.data_as(abi.dptr))
    return RigidTransform(R.reshape(3, 3), t)


def transform_from_twist(xi) -> RigidTransform:
    """proj/src/geometry.cpp:42-52 (reference evaluation order)."""
    x = np.ascontiguousarray(np.asarray(xi, np.float64).reshape(6))
    R, t = np.empty(9), np.empty(3)
    abi.synth_lib().lks_transform_from_twist(x.ctypes.data_as(abi.dptr), R.ctypes.data_as(abi.dptr),
                                             t.ctypes.data_as(abi.dptr))
    return RigidTransform(R.reshape(3, 3), t)


def compose(a: RigidTransform, b: RigidTransform) -> RigidTransform:
    """proj/src/geometry.cpp:8-11: b first, then a."""
    Ra, ta = np.ascontiguousarray(a.rotation, np.float64), np.ascontiguousarray(a.translation, np.float64)
    Rb, tb = np.ascontiguousarray(b.rotation, np.float64), np.ascontiguousarray(b.translation, np.float64)
    R, t = np.empty(9), np.empty(3)
    abi.synth_lib().lks_compose(Ra.ctypes.data_as(abi.dptr), ta.ctypes.data_as(abi.dptr), Rb.ctypes.data_as(abi.dptr),
                                tb.ctypes.data_as(abi.dptr), R.ctypes.data_as(abi.dptr), t.ctypes.data_as(abi.dptr))
    return RigidTransform(R.reshape(3, 3), t)


def inverse(a: RigidTransform) -> RigidTransform:
    Ra, ta = np.ascontiguousarray(a.rotation, np.float64), np.ascontiguousarray(a.translation, np.float64)
    R, t = np.empty(9), np.empty(3)
    abi.synth_lib().lks_inverse(Ra.ctypes.data_as(abi.dptr), ta.ctypes.data_as(abi.dptr), R.ctypes.data_as(abi.dptr),
                                t.ctypes.data_as(abi.dptr))
    return RigidTransform(R.reshape(3, 3), t)


def transformed(cloud: PointCloud, T: RigidTransform) -> PointCloud:
    """proj/src/geometry.cpp:105-114 (valid normals rotated, zero normals kept)."""
    L = abi.synth_lib()
    R = np.ascontiguousarray(T.rotation, np.float64)
    t = np.ascontiguousarray(T.translation, np.float64)
    n = cloud.size()
    out = np.empty((n, 3))
    L.lks_apply(R.ctypes.data_as(abi.dptr), t.ctypes.data_as(abi.dptr), cloud.positions.ctypes.data_as(abi.dptr), n,
                out.ctypes.data_as(abi.dptr))
    nrm = None
    if cloud.has_normals():
        nrm = np.empty((n, 3))
        L.lks_rotate(R.ctypes.data_as(abi.dptr), cloud.normals.ctypes.data_as(abi.dptr), n,
                     nrm.ctypes.data_as(abi.dptr))
        zero = ~cloud.normals.any(axis=1)
        nrm[zero] = cloud.normals[zero]
    return PointCloud(out, nrm)


def lattice_candidates(truth: RigidTransform, step_rad: float = 2.0 * math.pi / 180.0, step_m: float = 0.02,
                       half_rot: int = 3, half_trans: int = 1) -> Tuple[np.ndarray, int]:
    """Config A candidate list: truth o transform_from_twist(delta) over the
    lattice (a, b, g) in {-3..3} x step_rad, (x, y, z) in {-1, 0, 1} x step_m,
    lexicographic. Returns (C x 12 packed, index of the truth candidate)."""
    out = []
    truth_index = -1
    rr = range(-half_rot, half_rot + 1)
    tt = range(-half_trans, half_trans + 1)
    for a in rr:
        for b in rr:
            for g in rr:
                for x in tt:
                    for y in tt:
                        for z in tt:
                            if a == b == g == x == y == z == 0:
                                truth_index = len(out)
                            d = transform_from_twist([a * step_rad, b * step_rad, g * step_rad,
                                                      x * step_m, y * step_m, z * step_m])
                            out.append(compose(truth, d).packed())
    return np.ascontiguousarray(np.stack(out)), truth_index
