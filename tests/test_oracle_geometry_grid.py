"""Oracle pins: Kabsch / Jacobi SVD (proj/tests/test_geometry.cpp:84-140) and
grid queries against brute force (proj/tests/test_grid.cpp:14-125)."""
import math

import numpy as np
import pytest

from paper_1801_01572_b200 import synth


def _rigid_dist(Ra, ta, Rb, tb):
    return max(np.abs(Ra - Rb).max(), np.abs(ta - tb).max())


def test_kabsch_recovers_rigid_motion(oracle):
    # test_geometry.cpp:84-96 (RngStream(12, 0): transform then a 16-point cloud, 20 trials)
    for trial in range(20):
        T = synth.random_transform(12, trial)
        cloud = synth.random_cloud(16, 1200 + trial)
        dst = cloud.positions @ T.rotation.T + T.translation
        R, t = oracle.kabsch(cloud.positions, dst)
        assert _rigid_dist(R, t, T.rotation, T.translation) < 1e-9
        assert np.abs(R.T @ R - np.eye(3)).max() < 1e-9
        assert abs(np.linalg.det(R) - 1.0) < 1e-9


def test_kabsch_is_least_squares(oracle):
    # test_geometry.cpp:98-125
    T = synth.random_transform(13, 0, 0.5, 0.5)
    cloud = synth.random_cloud(200, 13, 1)
    rng = np.random.default_rng(13)
    dst = cloud.positions @ T.rotation.T + T.translation + 0.01 * rng.normal(size=(200, 3))
    R, t = oracle.kabsch(cloud.positions, dst)

    def cost(R_, t_):
        return float(((cloud.positions @ R_.T + t_ - dst) ** 2).sum())

    at_fit = cost(R, t)
    prng = np.random.default_rng(14)
    for _ in range(30):
        d = prng.uniform(-1e-3, 1e-3, size=6)
        D = synth.transform_from_twist(d)
        assert cost(D.rotation @ R, D.rotation @ t + D.translation) >= at_fit - 1e-12


def test_kabsch_rejects_degenerate_input(oracle):
    # test_geometry.cpp:127-140
    two = np.array([[0, 0, 0], [1, 0, 0]], float)
    with pytest.raises(oracle.OracleError) as e:
        oracle.kabsch(two, two)
    assert e.value.code == 3
    line = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0]], float)
    with pytest.raises(oracle.OracleError) as e:
        oracle.kabsch(line, line)
    assert e.value.code == 7
    coincident = np.tile([1.0, 2.0, 3.0], (4, 1))
    with pytest.raises(oracle.OracleError) as e:
        oracle.kabsch(coincident, coincident)
    assert e.value.code == 7


def test_jacobi_svd_reconstructs(oracle):
    rng = np.random.default_rng(3)
    for _ in range(200):
        A = rng.normal(size=(3, 3)) * rng.uniform(1e-3, 1e3)
        U, S, V = oracle.svd3(A)
        assert np.abs(U @ np.diag(S) @ V.T - A).max() < 1e-12 * max(1.0, np.abs(A).max())
        assert np.abs(U.T @ U - np.eye(3)).max() < 1e-13
        assert np.abs(V.T @ V - np.eye(3)).max() < 1e-13
        assert S[0] >= S[1] >= S[2] >= 0
        assert np.allclose(S, np.linalg.svd(A, compute_uv=False), rtol=1e-12, atol=1e-300)


def test_grid_index_floors(oracle):
    # test_grid.cpp:14-18 through nn_nearest on single-point grids
    g = oracle.SearchGrid(np.array([[0.05, 0.05, 0.05]]), 0.1)
    assert g.nn_within([0.05, 0.05, 0.05], 0.01)[0] == 0


def test_build_grid_rejects_bad_input(oracle):
    with pytest.raises(oracle.OracleError) as e:
        oracle.SearchGrid(np.zeros((0, 3)), 0.1)
    assert e.value.code == 2
    for cell in (0.0, -1.0):
        with pytest.raises(oracle.OracleError):
            oracle.SearchGrid(np.zeros((1, 3)), cell)


@pytest.mark.parametrize("cell", [0.02, 0.13, 0.5, 3.0])
def test_grid_queries_match_brute_force(oracle, cell):
    # test_grid.cpp:30-65 (600 points + 2 duplicates of point 17, 200 queries)
    cloud = synth.random_cloud(600, 21, int(cell * 100)).positions
    cloud = np.vstack([cloud, cloud[17], cloud[17]])
    g = oracle.SearchGrid(cloud, cell)
    rng = np.random.default_rng(int(cell * 1000))
    for q in rng.uniform(-1.4, 1.4, size=(200, 3)):
        for d_max in (0.05, 0.2, 1.0):
            fast = g.nn_within(q, d_max)
            slow = oracle.bf_nn_within(cloud, q, d_max)
            assert (fast is None) == (slow is None)
            if fast:
                assert fast[0] == slow[0]
                assert fast[1] == pytest.approx(slow[1], rel=1e-12)
        i, d = g.nn_nearest(q)
        dd = np.linalg.norm(cloud - q, axis=1)
        assert i == int(np.argmin(dd))
        assert d == pytest.approx(dd.min(), rel=1e-12)
        for radius in (0.1, 0.4):
            assert g.radius_search(q, radius) == sorted(np.nonzero(((cloud - q) ** 2).sum(1) <= radius * radius)[0].tolist())


def test_far_queries_stay_exact(oracle):
    # test_grid.cpp:67-76
    cloud = synth.random_cloud(50, 22).positions
    g = oracle.SearchGrid(cloud, 0.25)
    far = np.array([40.0, -35.0, 12.0])
    i, d = g.nn_nearest(far)
    assert i == int(np.argmin(np.linalg.norm(cloud - far, axis=1)))
    assert g.nn_within(far, 1.0) is None


def test_radius_search_inclusive(oracle):
    # test_grid.cpp:94-100
    g = oracle.SearchGrid(np.array([[0, 0, 0], [1, 0, 0]], float), 0.3)
    assert g.radius_search([0, 0, 0], 1.0) == [0, 1]


def test_feature_cache_exhaustive_ties_lowest(oracle):
    # test_grid.cpp:113-125
    rng = np.random.default_rng(23)
    src = rng.uniform(0, 100, size=(300, 33)).astype(np.float32)
    tgt = rng.uniform(0, 100, size=(250, 33)).astype(np.float32)
    tgt[190] = tgt[40]
    src[7] = tgt[40]
    got = oracle.feature_nn_cache(src, tgt)
    d2 = ((src[:, None, :].astype(np.float64) - tgt[None, :, :].astype(np.float64)) ** 2).sum(-1)
    assert (got == d2.argmin(1)).all()
    assert got[7] == 40
    for threads in (1, 4, 16):
        assert (oracle.feature_nn_cache(src, tgt, threads) == got).all()
    with pytest.raises(oracle.OracleError):
        oracle.feature_nn_cache(np.zeros((0, 33), np.float32), tgt)
