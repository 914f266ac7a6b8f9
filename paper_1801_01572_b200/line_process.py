"""Line-process weight of a loop edge, the host-side
consumer of ``edge_info`` / ``verify_batch``: whether a verified loop closure
is kept is decided from its information matrix and the poses, on the host
(``include/loopkit_b200.h`` ``lk_edge_residual`` / ``lk_update_weight`` /
``lk_loop_weights``).

- ``edge_residual``  -- ``proj/src/line_process.cpp:35-40``: f = xi^T Lambda xi,
  xi = twist(rel * T_j^-1 * T_i) (``geometry.cpp:28-40``); RotationTooLarge at
  a residual rotation of pi/2 or more.
- ``update_weight``  -- ``line_process.cpp:42-46``: (mu / (mu + max(f, 0)))^2
  clamped to [0, 1]; 0 for mu <= 0.
- ``loop_weights``   -- ``line_process.cpp:52-67, 100-103``: per loop edge,
  mu = mu_tau * pair_count, the small-angle gate of ``loop_residual`` (weight
  0 beyond pi/2) and the accept label weight >= reject_threshold, at the given
  poses (the pose-graph optimisation around it is out of this tier's scope).
"""
from __future__ import annotations

import ctypes as C
from typing import Sequence, Tuple

import numpy as np

from . import abi
from .errors import check

__all__ = ["edge_residual", "update_weight", "loop_weights"]


def _t12(T) -> np.ndarray:
    return np.ascontiguousarray(np.concatenate([np.asarray(T.rotation, np.float64).reshape(9),
                                                np.asarray(T.translation, np.float64).reshape(3)]))


def _info36(info) -> np.ndarray:
    m = getattr(info, "info", info)
    return np.ascontiguousarray(np.asarray(m, np.float64).reshape(36))


def edge_residual(t_i, t_j, rel, info) -> float:
    """line_process.cpp:35-40 (``info``: an EdgeInfo or a 6x6 array)."""
    f = C.c_double()
    a, b, r, m = _t12(t_i), _t12(t_j), _t12(rel), _info36(info)
    check(abi.lib().lk_edge_residual(a.ctypes.data_as(abi.dptr), b.ctypes.data_as(abi.dptr),
                                     r.ctypes.data_as(abi.dptr), m.ctypes.data_as(abi.dptr), C.byref(f)))
    return f.value


def update_weight(f: float, mu: float) -> float:
    """line_process.cpp:42-46."""
    return float(abi.lib().lk_update_weight(float(f), float(mu)))


def loop_weights(pose_i: Sequence, pose_j: Sequence, rel: Sequence, infos: Sequence, mu_tau: float = 0.2,
                 reject_threshold: float = 0.25) -> Tuple[np.ndarray, np.ndarray]:
    """Weights and accept labels of loop edges at the given poses; ``infos``
    are EdgeInfo objects (e.g. ``VerifyResult.info``), whose pair_count sets
    mu = mu_tau * pair_count (LineProcessOptions, line_process.hpp:24-31)."""
    n = len(infos)
    Ti = np.ascontiguousarray(np.stack([_t12(t) for t in pose_i]) if n else np.zeros((1, 12)))
    Tj = np.ascontiguousarray(np.stack([_t12(t) for t in pose_j]) if n else np.zeros((1, 12)))
    Tr = np.ascontiguousarray(np.stack([_t12(t) for t in rel]) if n else np.zeros((1, 12)))
    M = np.ascontiguousarray(np.stack([_info36(e) for e in infos]) if n else np.zeros((1, 36)))
    cnt = np.ascontiguousarray(np.array([int(e.pair_count) for e in infos] or [0], dtype=np.int64))
    w = np.zeros(max(n, 1))
    acc = np.zeros(max(n, 1), dtype=np.int32)
    check(abi.lib().lk_loop_weights(n, Ti.ctypes.data_as(abi.dptr), Tj.ctypes.data_as(abi.dptr),
                                    Tr.ctypes.data_as(abi.dptr), M.ctypes.data_as(abi.dptr),
                                    cnt.ctypes.data_as(C.POINTER(C.c_int64)), float(mu_tau), float(reject_threshold),
                                    w.ctypes.data_as(abi.dptr), acc.ctypes.data_as(C.POINTER(C.c_int32))))
    return w[:n], acc[:n].astype(bool)
