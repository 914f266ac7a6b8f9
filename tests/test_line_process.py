"""Line-process weight of a loop edge (row a11; paper_1801_01572_b200/line_process.py
over lk_edge_residual / lk_update_weight / lk_loop_weights): the reference's
own test cases (proj/tests/test_line_process.cpp:42-65, 111-126) and the
definition restated with numpy. Host-only: no GPU."""
import math

import numpy as np
import pytest

import paper_1801_01572_b200 as lk
from paper_1801_01572_b200 import synth


def _isotropic(kappa):
    # test_line_process.cpp:30-38: Lambda = kappa I, pair_count = kappa
    return lk.EdgeInfo(kappa * np.eye(6), int(kappa))


def _twist(T):
    # geometry.cpp:28-40, restated
    R = T.rotation
    assert math.acos(min(max((np.trace(R) - 1.0) / 2.0, -1.0), 1.0)) < math.pi / 2
    beta = math.asin(min(max(R[0, 2], -1.0), 1.0))
    return np.array([math.atan2(-R[1, 2], R[2, 2]), beta, math.atan2(-R[0, 1], R[0, 0]), *T.translation])


def _numeric_weight(f, mu):
    # the 1-D energy l f + mu (sqrt l - 1)^2 minimised on a fine grid, then refined
    ls = np.linspace(0.0, 1.0, 200001)
    e = ls * f + mu * (np.sqrt(ls) - 1.0) ** 2
    return float(ls[np.argmin(e)])


def test_update_weight_reference_cases():
    for mu in (0.5, 1.0, 10.0, 250.0):
        for f in (0.0, 1e-4, 0.3, 1.0, mu, 5.0 * mu, 100.0 * mu):
            w = lk.update_weight(f, mu)
            assert 0.0 <= w <= 1.0
            assert abs(w - _numeric_weight(f, mu)) < 2e-5  # grid resolution of the restated minimiser
            assert w == (mu / (mu + f)) ** 2
    assert lk.update_weight(0.0, 3.0) == 1.0
    assert lk.update_weight(1.0, 0.0) == 0.0
    assert lk.update_weight(1.0, -2.0) == 0.0
    assert lk.update_weight(-5.0, 2.0) == 1.0  # max(f, 0)
    assert lk.update_weight(5.0, 1.0) == pytest.approx(1.0 / 36.0, rel=1e-12)
    assert lk.update_weight(5.0, 1.0) < 0.25
    assert lk.update_weight(1.0, 1.0) == pytest.approx(0.25, rel=1e-12)


def test_edge_residual_is_the_mahalanobis_norm_of_the_residual_twist():
    ti = synth.random_transform(72, 0, 0.3, 0.5)
    tj = synth.random_transform(72, 1, 0.3, 0.5)
    rel = synth.compose(synth.inverse(ti), tj)  # exactly consistent
    info = _isotropic(7.0)
    assert lk.edge_residual(ti, tj, rel, info) == pytest.approx(0.0, abs=1e-12)
    ti2 = synth.compose(ti, synth.transform_from_twist([0.01, -0.02, 0.015, 0.05, -0.03, 0.02]))
    f = lk.edge_residual(ti2, tj, rel, info)
    xi = _twist(synth.compose(rel, synth.compose(synth.inverse(tj), ti2)))
    assert f == pytest.approx(float(xi @ (info.info @ xi)), rel=1e-12)
    assert f > 0.0
    # an anisotropic information matrix weights the components
    A = np.diag([1.0, 2.0, 3.0, 4.0, 5.0, 6.0])
    A[0, 3] = A[3, 0] = 0.5
    assert lk.edge_residual(ti2, tj, rel, A) == pytest.approx(float(xi @ (A @ xi)), rel=1e-12)


def test_edge_residual_rotation_too_large():
    I = lk.RigidTransform()
    half_turn = synth.transform_from_twist([0.0, 0.0, math.pi * 0.6, 0.0, 0.0, 0.0])
    with pytest.raises(lk.RotationTooLarge):
        lk.edge_residual(half_turn, I, I, np.eye(6))


def test_loop_weights_labels_and_the_small_angle_gate():
    I = lk.RigidTransform()
    good = synth.transform_from_twist([0.001, 0.0, 0.0, 0.002, 0.0, 0.0])
    bad = synth.transform_from_twist([0.2, 0.1, 0.0, 0.5, 0.0, 0.0])
    huge = synth.transform_from_twist([0.0, 0.0, 2.0, 0.0, 0.0, 0.0])
    infos = [_isotropic(100.0), _isotropic(100.0), _isotropic(100.0), lk.EdgeInfo(np.eye(6), 0)]
    w, acc = lk.loop_weights([good, bad, huge, good], [I] * 4, [I] * 4, infos, mu_tau=0.2, reject_threshold=0.25)
    for k in (0, 1):
        f = lk.edge_residual([good, bad][k], I, I, infos[k])
        assert w[k] == lk.update_weight(f, 0.2 * infos[k].pair_count)
    assert acc[0] and not acc[1]
    assert w[2] == 0.0 and not acc[2]  # beyond pi/2: loop_residual -> weight 0
    assert w[3] == 0.0 and not acc[3]  # vacuous edge: mu = 0
    w0, acc0 = lk.loop_weights([], [], [], [])
    assert w0.shape == (0,) and acc0.shape == (0,)
