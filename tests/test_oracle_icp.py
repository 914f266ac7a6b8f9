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


def test_oracle_estimate_normals_reference_cases(oracle):
    """preprocess.cpp:61-96 restated; the reference's own cases
    (proj/tests/test_preprocess.cpp:77-122)."""
    P = np.array([[0.05 * i, 0.05 * j, 0.0] for i in range(20) for j in range(20)])
    N = oracle.estimate_normals(P, 0.12, (0.5, 0.5, 2.0))
    assert np.allclose(np.linalg.norm(N, axis=1), 1.0, atol=1e-9)
    assert np.allclose(N[:, 2], 1.0, atol=1e-6)
    assert np.allclose(oracle.estimate_normals(P, 0.12, (0.5, 0.5, -2.0))[:, 2], -1.0, atol=1e-6)
    c = np.array([[0, 0, 0], [0.01, 0, 0], [0.02, 0, 0], [10, 10, 10.0]])
    N = oracle.estimate_normals(c, 0.05, (0, 0, 1))
    assert np.linalg.norm(N[3]) == 0.0
    assert abs(np.linalg.norm(N[0]) - 1.0) < 1e-9 and abs(N[0, 0]) < 1e-9
    rng = np.random.default_rng(32)
    R = rng.uniform(-1, 1, size=(400, 3))
    base = oracle.estimate_normals(R, 0.3, threads=1)
    for t in (2, 4, 16):
        assert np.array_equal(oracle.estimate_normals(R, 0.3, threads=t), base)
    # against a plain eigen-decomposition: same normal line (sign is the viewpoint's)
    for i in range(0, 400, 37):
        nb = np.where(np.sum((R - R[i]) ** 2, axis=1) <= 0.09)[0]
        if len(nb) < 3:
            continue
        d = R[nb] - R[nb].mean(axis=0)
        w, V = np.linalg.eigh(d.T @ d)
        if w[1] - w[0] > 1e-6 * w[2]:
            assert abs(abs(V[:, 0] @ base[i]) - 1.0) < 1e-9
