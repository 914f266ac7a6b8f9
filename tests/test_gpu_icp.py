"""GPU ICP (lk_icp.cu) against the frozen ICP oracle: transform, iteration
count, correspondences, rmse and the per-iteration history bit for bit (the
device reduces in the oracle's tree order and solves / updates with the same
IEEE operations), on the FP32 fine-list path and the FP64-only path."""
import numpy as np
import pytest

import paper_1801_01572_b200 as lk
from paper_1801_01572_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if lk.device_count() == 0:
        pytest.fail("no CUDA device visible: -m gpu tests must run on the B200 box")


def _perturbed(T, xi):
    return synth.compose(synth.transform_from_twist(xi), T)


def _check_same(oracle, pair, T0, dmax, iters, eps):
    R, t, res, hist = oracle.icp_point_to_plane(pair.source.positions, pair.target.positions, pair.target.normals,
                                                T0.rotation, T0.translation, dmax, iters, eps)
    dev = lk.icp_point_to_plane(pair.source, pair.target, T0,
                                lk.IcpParams(max_correspondence_distance=dmax, max_iterations=iters,
                                             convergence_eps=eps))
    assert dev.iterations == res.iterations
    assert dev.converged == bool(res.converged)
    assert dev.correspondences == res.correspondences
    assert dev.rmse == res.rmse
    assert np.array_equal(dev.transform.rotation, R)
    assert np.array_equal(dev.transform.translation, t)
    assert np.array_equal(dev.history, hist[: len(dev.history)])
    return dev


@pytest.mark.parametrize("fp64_only", [False, True])  # True: infinite band, every shell in FP64
def test_icp_submaps_match_oracle(oracle, monkeypatch, fp64_only):
    if fp64_only:
        monkeypatch.setenv("LK_FP64_ONLY", "1")
    pair = synth.submap_pair(views=4, stride=8)
    T0 = _perturbed(pair.truth, [0.02, -0.015, 0.01, 0.02, -0.01, 0.015])
    dev = _check_same(oracle, pair, T0, 0.05, 30, 1e-10)
    assert dev.converged


def test_icp_noise_free_and_max_iterations(oracle):
    pair = synth.surface_pair(seed=1, density=600.0, noise=0.0)
    T0 = _perturbed(pair.truth, [0.01, -0.012, 0.008, 0.01, -0.006, 0.008])
    dev = _check_same(oracle, pair, T0, 0.05, 40, 1e-12)
    assert np.abs(dev.transform.rotation - pair.truth.rotation).max() < 1e-9
    _check_same(oracle, pair, T0, 0.05, 3, 0.0)  # stops at max_iterations, unconverged
    _check_same(oracle, pair, T0, 0.03, 0, 1e-12)


def test_icp_errors():
    pair = synth.surface_pair(seed=2, density=200.0, noise=0.0)
    far = lk.PointCloud(pair.source.positions + 100.0)
    with pytest.raises(lk.NoCorrespondences):
        lk.icp_point_to_plane(far, pair.target, lk.RigidTransform(np.eye(3), np.zeros(3)))
    with pytest.raises(lk.MissingNormals):
        lk.icp_point_to_plane(pair.source, lk.PointCloud(pair.target.positions),
                              lk.RigidTransform(np.eye(3), np.zeros(3)))
    with pytest.raises(lk.EmptyCloud):
        lk.icp_point_to_plane(lk.PointCloud(np.zeros((0, 3))), pair.target, lk.RigidTransform(np.eye(3), np.zeros(3)))


def test_icp_exact_ties_take_the_lower_index(oracle):
    """Every target point twice, the copy (higher index) with a different
    normal: each query meets an exact distance tie, which the reference's
    (d2, index) order gives to the original. Exercises the band re-scan of the
    warp-cooperative ring walk."""
    pair = synth.surface_pair(seed=4, density=600.0, noise=0.002)
    P, N = pair.target.positions, pair.target.normals
    tilt = synth.transform_from_twist([0.3, -0.2, 0.1, 0.0, 0.0, 0.0]).rotation
    tgt = lk.PointCloud(np.vstack([P, P]), np.vstack([N, N @ tilt.T]))
    dup = synth.RegistrationPair(pair.source, tgt, pair.truth)
    T0 = _perturbed(pair.truth, [0.01, -0.012, 0.008, 0.01, -0.006, 0.008])
    dev = _check_same(oracle, dup, T0, 0.05, 12, 1e-10)
    ref = _check_same(oracle, pair, T0, 0.05, 12, 1e-10)  # the original normals decide
    assert dev.iterations == ref.iterations and np.array_equal(dev.transform.rotation, ref.transform.rotation)


def test_icp_scattered_queries_and_outliers(oracle):
    """A source with a fifth of its points scattered far and wide (misses, and
    queries many cells outside the grid) and in shuffled order: warps whose
    queries span more than the cooperative window fall back to per-lane walks;
    the result is still the oracle's bit for bit."""
    pair = synth.surface_pair(seed=5, density=500.0, noise=0.003)
    rng = np.random.default_rng(11)
    src = pair.source.positions.copy()
    k = len(src) // 5
    idx = rng.choice(len(src), k, replace=False)
    src[idx] = rng.uniform(-6.0, 6.0, size=(k, 3))
    src = src[rng.permutation(len(src))]
    scattered = synth.RegistrationPair(lk.PointCloud(src), pair.target, pair.truth)
    T0 = _perturbed(pair.truth, [0.01, 0.01, -0.008, 0.005, 0.01, -0.004])
    _check_same(oracle, scattered, T0, 0.05, 10, 1e-10)


def test_icp_singular_plane_stops_like_the_oracle(oracle):
    """A plane against a plane (every normal +z): in-plane translation and the
    rotation about z are unobservable, the LDL^T meets a zero pivot and the
    run stops where the oracle stops, with the same history."""
    g = np.array([[0.02 * a, 0.02 * b, 0.0] for a in range(40) for b in range(40)])
    n = np.tile([0.0, 0.0, 1.0], (len(g), 1))
    src = lk.PointCloud(g + np.array([0.003, -0.002, 0.01]))
    tgt = lk.PointCloud(g, n)
    pair = synth.RegistrationPair(src, tgt, lk.RigidTransform())
    dev = _check_same(oracle, pair, lk.RigidTransform(), 0.05, 10, 1e-12)
    assert not dev.converged
