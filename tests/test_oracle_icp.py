"""ICP oracle (north-star item 4; no reference -- SPEC.md:332): the frozen
spec of oracle/lk_oracle.cpp "ICP point-to-plane" pinned by properties:
exact recovery on noise-free data, monotone convergence, error cases."""
import math

import numpy as np
import pytest

from paper_1801_01572_b200 import synth


def _perturbed(T, xi):
    return synth.compose(synth.transform_from_twist(xi), T)


def test_icp_recovers_truth_on_noise_free_surfaces(oracle):
    pair = synth.surface_pair(seed=1, density=600.0, noise=0.0)
    T0 = _perturbed(pair.truth, [0.01, -0.012, 0.008, 0.01, -0.006, 0.008])
    R, t, res, hist = oracle.icp_point_to_plane(pair.source.positions, pair.target.positions, pair.target.normals,
                                                T0.rotation, T0.translation, 0.05, 40, 1e-12)
    assert res.converged == 1
    assert np.abs(R - pair.truth.rotation).max() < 1e-9
    assert np.abs(t - pair.truth.translation).max() < 1e-9
    assert res.rmse < 1e-9
    assert res.correspondences == pair.source.size()


def test_icp_rmse_decreases_on_submaps(oracle):
    pair = synth.submap_pair(views=4, stride=8)
    T0 = _perturbed(pair.truth, [0.02, -0.015, 0.01, 0.02, -0.01, 0.015])
    R, t, res, hist = oracle.icp_point_to_plane(pair.source.positions, pair.target.positions, pair.target.normals,
                                                T0.rotation, T0.translation, 0.05, 30, 1e-10)
    assert res.converged == 1 and 2 <= res.iterations < 30
    h = hist[: res.iterations]
    assert h[0, 1] > h[-1, 1]  # rmse falls
    assert all(h[k + 1, 2] < h[k, 2] for k in range(3))  # steps shrink
    # the refined pose is within the noise floor of the truth
    dR = pair.truth.rotation.T @ R
    assert math.acos(max(-1.0, min(1.0, (np.trace(dR) - 1) / 2))) < 2e-3
    assert np.linalg.norm(t - pair.truth.translation) < 5e-3


def test_icp_errors(oracle):
    pair = synth.surface_pair(seed=2, density=200.0, noise=0.0)
    far = pair.source.positions + 100.0
    with pytest.raises(oracle.OracleError) as e:
        oracle.icp_point_to_plane(far, pair.target.positions, pair.target.normals, np.eye(3), np.zeros(3), 0.05)
    assert e.value.code == 6  # NoCorrespondences
    with pytest.raises(oracle.OracleError) as e:
        oracle.icp_point_to_plane(pair.source.positions, pair.target.positions, None, np.eye(3), np.zeros(3), 0.05)
    assert e.value.code == 5  # MissingNormals
    with pytest.raises(oracle.OracleError):
        oracle.icp_point_to_plane(pair.source.positions, pair.target.positions, pair.target.normals, np.eye(3),
                                  np.zeros(3), 0.0)


def test_icp_zero_iterations_is_identity(oracle):
    pair = synth.surface_pair(seed=3, density=200.0, noise=0.0)
    T0 = _perturbed(pair.truth, [0.01, 0, 0, 0, 0, 0])
    R, t, res, hist = oracle.icp_point_to_plane(pair.source.positions, pair.target.positions, pair.target.normals,
                                                T0.rotation, T0.translation, 0.05, 0)
    assert res.iterations == 0 and np.array_equal(R, T0.rotation) and np.array_equal(t, T0.translation)
