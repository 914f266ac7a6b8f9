"""GPU parity: the sm_100a path through the C ABI against the CPU oracle.

Bar: winner index, inlier counts, found/not
found and all HypothesisStats counters bit-exact; fitness and the transform
bit-exact too (the device reproduces the oracle's FP64 operation order with
no FMA). edge_info: pair_count exact, information matrix within 1e-9 rel.
"""
import math

import numpy as np
import pytest

import paper_1801_01572_b200 as lk
from paper_1801_01572_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if lk.device_count() == 0:
        pytest.fail("no CUDA device visible: -m gpu tests must run on the B200 box")


@pytest.fixture(scope="module")
def pair1():
    return synth.synth_registration_pair(1)


@pytest.fixture(scope="module")
def prepared1(oracle, pair1):
    p = oracle.params(hypothesis_count=100_000, seed=1)
    ctx = oracle.Context.prepare(pair1.source.positions, pair1.source.normals, pair1.target.positions,
                                 pair1.target.normals, p)
    return ctx, ctx.get()


def _assert_same_result(dev, orc, dev_stats=None, orc_stats=None):
    assert (dev is not None) == orc.found
    if orc.found:
        assert dev.hypothesis_index == orc.hypothesis_index
        assert dev.inliers == orc.inliers
        assert dev.inlier_ratio == orc.inlier_ratio
        assert dev.fitness == orc.fitness  # bitwise: same sequential FP64 sum
        assert np.array_equal(dev.transform.rotation, orc.R)
        assert np.array_equal(dev.transform.translation, orc.t)
    if dev_stats is not None:
        for k in ("sampled", "prerejected", "degenerate", "evaluated", "qualified", "w_ref"):
            assert getattr(dev_stats, k) == orc_stats[k], k


def test_feature_nn_cache_matches_oracle(prepared1, oracle):
    _, c = prepared1
    got = lk.feature_nn_cache(c["src_feat"], c["tgt_feat"])
    assert np.array_equal(got, c["cache"])
    # exact duplicate -> lowest index (test_grid.cpp:113-125)
    rng = np.random.default_rng(23)
    src = rng.uniform(0, 100, size=(300, 33)).astype(np.float32)
    tgt = rng.uniform(0, 100, size=(250, 33)).astype(np.float32)
    tgt[190] = tgt[40]
    src[7] = tgt[40]
    assert np.array_equal(lk.feature_nn_cache(src, tgt), oracle.feature_nn_cache(src, tgt))


@pytest.mark.parametrize("fp64_only", ["0", "1"])
def test_feature_nn_near_ties(oracle, monkeypatch, fp64_only):
    # targets one ulp away from a source feature, exact duplicates, zero features:
    # the FP32 pre-match must hand every near-tie to the exact FP64 resolution
    monkeypatch.setenv("LK_FP64_ONLY", fp64_only)
    rng = np.random.default_rng(5)
    src = rng.uniform(0, 200, size=(700, 33)).astype(np.float32)
    tgt = rng.uniform(0, 200, size=(900, 33)).astype(np.float32)
    for k in range(0, 600, 3):
        t = src[k].copy()
        tgt[(7 * k) % 900] = t
        t2 = t.copy()
        t2[k % 33] = np.nextafter(t2[k % 33], np.float32(1e9))
        tgt[(7 * k + 1) % 900] = t2
        t3 = t.copy()
        t3[(k + 5) % 33] = np.nextafter(t3[(k + 5) % 33], np.float32(-1e9))
        tgt[(7 * k + 2) % 900] = t3
    src[650:] = 0.0
    tgt[100] = 0.0
    tgt[400] = 0.0
    assert np.array_equal(lk.feature_nn_cache(src, tgt), oracle.feature_nn_cache(src, tgt))


def test_eval_grid_build_matches_oracle(pair1, oracle):
    t = pair1.target
    g = lk.build_eval_grid(t, 0.075)
    og = oracle.EvalGrid(t.positions, t.normals, 0.075)
    assert np.array_equal(g.origin, og.origin)
    assert g.dims == og.dims and g.ncells == og.ncells
    a, b = g.download(), og.arrays()
    for k in ("start", "index", "slot_position", "slot_normal", "near_occupied"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("units", ["auto", "1", "0"])  # scorer: by candidate count / round units / CTA per candidate
@pytest.mark.parametrize("seed,H", [(1, 100_000), (7, 20_000), (3, 50_000)])
def test_run_hypotheses_matches_oracle(prepared1, oracle, monkeypatch, seed, H, units):
    if units != "auto":
        monkeypatch.setenv("LK_SCORE_UNITS", units)
    octx, c = prepared1
    params = lk.RegistrationParams(hypothesis_count=H, seed=seed)
    ctx = lk.registration_context(lk.PointCloud(c["src"], c["src_n"]), lk.PointCloud(c["tgt"], c["tgt_n"]),
                                  c["cache"], params)
    st = lk.HypothesisStats()
    dev = lk.run_hypotheses(ctx, params, st)
    orc, ost = octx.run(oracle.params_from(params))
    _assert_same_result(dev, orc, st, ost)
    assert st.evals_executed >= st.w_ref


@pytest.mark.parametrize("kw", [
    dict(normal_angle_max=8.0 * math.pi / 180.0, min_inlier_ratio=0.05),   # many gate decisions near cos_max
    dict(normal_angle_max=75.0 * math.pi / 180.0),
    dict(max_fitness=0.0009, min_inlier_ratio=0.1),                        # qualification near the fitness bar
    dict(min_inlier_ratio=0.0),                                            # zero-inlier candidates qualify
])
def test_run_hypotheses_params_match_oracle(prepared1, oracle, kw):
    # the scorer's FP32 normal gate, the order-bound qualification and the
    # exact chains on demand must reproduce the reference's decisions
    octx, c = prepared1
    params = lk.RegistrationParams(hypothesis_count=60_000, seed=5, **kw)
    ctx = lk.registration_context(lk.PointCloud(c["src"], c["src_n"]), lk.PointCloud(c["tgt"], c["tgt_n"]),
                                  c["cache"], params)
    st = lk.HypothesisStats()
    dev = lk.run_hypotheses(ctx, params, st)
    orc, ost = octx.run(oracle.params_from(params))
    _assert_same_result(dev, orc, st, ost)


def test_prepare_and_register_global_match_oracle(pair1, oracle):
    params = lk.RegistrationParams(hypothesis_count=100_000, seed=1)
    ctx = lk.prepare_registration(pair1.source, pair1.target, params)
    src, tgt, cache, sf, tf = ctx.download()
    octx = oracle.Context.prepare(pair1.source.positions, pair1.source.normals, pair1.target.positions,
                                  pair1.target.normals, oracle.params_from(params))
    c = octx.get()
    assert np.array_equal(src.positions, c["src"]) and np.array_equal(src.normals, c["src_n"])
    assert np.array_equal(tgt.positions, c["tgt"]) and np.array_equal(tgt.normals, c["tgt_n"])
    assert np.array_equal(sf, c["src_feat"]) and np.array_equal(tf, c["tgt_feat"])
    assert np.array_equal(cache, c["cache"])
    st = lk.HypothesisStats()
    dev = lk.register_global(pair1.source, pair1.target, params, st)
    orc, ost = octx.run(oracle.params_from(params))
    _assert_same_result(dev, orc, st, ost)
    # test_registration.cpp:162-179 on the device result
    Rerr = pair1.truth.rotation.T @ dev.transform.rotation
    assert math.acos(max(-1.0, min(1.0, (np.trace(Rerr) - 1) / 2))) < 3 * math.pi / 180
    assert np.linalg.norm(pair1.truth.rotation.T @ (dev.transform.translation - pair1.truth.translation)) < 0.05
    assert st.prerejected + st.degenerate + st.evaluated == st.sampled == 100_000


def test_device_estimate_normals_matches_oracle(oracle):
    # estimate_normals (preprocess.cpp:61-96): radius_search neighbours, the
    # sequential mean / covariance sums, the restated Eigen eigensolver, the
    # viewpoint orientation -- bitwise against the oracle
    rng = np.random.default_rng(32)
    plane = np.array([[0.05 * i, 0.05 * j, 0.0] for i in range(20) for j in range(20)])
    frame = lk.voxel_downsample(synth.depth_frame_pair().target, 0.02).positions
    cases = [(rng.uniform(-1, 1, size=(400, 3)), 0.3, (0.0, 0.0, 0.0)), (plane, 0.12, (0.5, 0.5, 2.0)),
             (plane, 0.12, (0.5, 0.5, -2.0)), (np.array([[0, 0, 0], [0.01, 0, 0], [0.02, 0, 0], [10, 10, 10.0]]), 0.05,
                                                (0.0, 0.0, 1.0)), (frame, 0.1, (0.0, 0.0, 0.0))]
    # degenerate neighbourhoods: coincident points (zero covariance), a line
    # (two zero eigenvalues), exact ties in the eigenvalues of a regular grid
    dup = np.vstack([np.zeros((5, 3)), np.array([[0.5, 0.0, 0.0], [0.0, 0.0, 3.0]])])
    line = np.array([[0.01 * k, 0.0, 0.0] for k in range(12)])
    cube = np.array([[0.05 * a, 0.05 * b, 0.05 * c] for a in range(4) for b in range(4) for c in range(4)])
    cases += [(dup, 0.1, (1.0, 2.0, 3.0)), (line, 0.05, (0.0, 1.0, 0.0)), (cube, 0.06, (0.0, 0.0, 0.0))]
    # above the brute-force size the SearchGrid neighbour lists are used
    big = lk.voxel_downsample(synth.depth_frame_pair().target, 0.008).positions
    assert len(big) > 24576
    cases.append((big, 0.03, (0.0, 0.0, 0.0)))
    for xyz, r, vp in cases:
        dev = lk.estimate_normals(lk.PointCloud(xyz), r, vp).normals
        assert np.array_equal(dev, oracle.estimate_normals(xyz, r, vp)), (len(xyz), r)
    assert np.allclose(lk.estimate_normals(lk.PointCloud(plane), 0.12, (0.5, 0.5, 2.0)).normals[:, 2], 1.0)
    with pytest.raises(lk.EmptyCloud):
        lk.estimate_normals(lk.PointCloud(np.zeros((0, 3))), 0.1)


def test_normal_less_clouds_register_like_the_oracle(pair1, oracle):
    # registration.cpp:232-237: clouds given without normals get
    # estimate_normals(normal_radius, origin) after downsampling
    params = lk.RegistrationParams(hypothesis_count=60_000, seed=2)
    S, T = lk.PointCloud(pair1.source.positions), lk.PointCloud(pair1.target.positions)
    ctx = lk.prepare_registration(S, T, params)
    src, tgt, cache, sf, tf = ctx.download()
    octx = oracle.Context.prepare(S.positions, None, T.positions, None, oracle.params_from(params))
    c = octx.get()
    assert np.array_equal(src.normals, c["src_n"]) and np.array_equal(tgt.normals, c["tgt_n"])
    assert np.array_equal(sf, c["src_feat"]) and np.array_equal(tf, c["tgt_feat"])
    assert np.array_equal(cache, c["cache"])
    st = lk.HypothesisStats()
    dev = lk.register_global(S, T, params, st)
    orc, ost = octx.run(oracle.params_from(params))
    _assert_same_result(dev, orc, st, ost)


def test_device_prepare_helpers_match_oracle(oracle):
    # device voxel_downsample (preprocess.cpp:14-59) and FPFH (fpfh.cpp:57-141), bitwise
    pair = synth.synth_registration_pair(4)
    for cloud in (pair.source, pair.target):
        d = lk.voxel_downsample(cloud, 0.05)
        ox, on = oracle.voxel_downsample(cloud.positions, cloud.normals, 0.05)
        assert np.array_equal(d.positions, ox) and np.array_equal(d.normals, on)
        f = lk.compute_fpfh(d, 0.25)
        fo = oracle.compute_fpfh(ox, on, 0.25)
        assert np.array_equal(f, fo)


@pytest.mark.parametrize("n,half", [(1500, 0.2), (3000, 1.5)])
def test_device_fpfh_dense_and_sparse_match_oracle(oracle, n, half):
    # (1500 points in a 0.4 m box: > 192 neighbours within 0.25 m -- the
    # slot table overflows and the exact two-pass fill runs) and a sparse cloud
    c = synth.random_cloud(n, 77, 3, -half, half, with_normals=True)
    f = lk.compute_fpfh(c, 0.25)
    fo = oracle.compute_fpfh(c.positions, c.normals, 0.25)
    assert np.array_equal(f, fo)


def test_device_downsample_full_frame_matches_oracle(oracle):
    # 307k-point depth frame: dense voxels (hundreds of points each), zero normals mixed in
    pair = synth.depth_frame_pair()
    src = pair.source
    nrm = src.normals.copy()
    nrm[::97] = 0.0
    cloud = lk.PointCloud(src.positions, nrm)
    for leaf in (0.05, 0.02):
        d = lk.voxel_downsample(cloud, leaf)
        ox, on = oracle.voxel_downsample(cloud.positions, cloud.normals, leaf)
        assert np.array_equal(d.positions, ox) and np.array_equal(d.normals, on)
    # FPFH above the brute-force size limit takes the SearchGrid path
    assert d.size() > 24576
    f = lk.compute_fpfh(d, 0.08)
    fo = oracle.compute_fpfh(ox, on, 0.08)
    assert np.array_equal(f, fo)
    bad = src.normals.copy()
    bad[5] *= 1.1
    with pytest.raises(lk.MissingNormals):
        lk.voxel_downsample(lk.PointCloud(src.positions, bad), 0.05)


@pytest.mark.parametrize("cluster", [1000, 1024, 1025, 5000])
def test_device_downsample_voxel_group_sizes(oracle, cluster):
    # one voxel holding 1000-5000 of the points among sparse ones: members in
    # input order through the stable radix sort, sums in the reference's order
    rng = np.random.default_rng(cluster)
    spread = rng.uniform(-2.0, 2.0, size=(20_000, 3))
    dense = 0.4 + rng.uniform(0.0, 0.049, size=(cluster, 3))  # one 0.05 voxel
    pos = np.concatenate([spread[:7_000], dense, spread[7_000:]])
    nrm = rng.normal(size=pos.shape)
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    cloud = lk.PointCloud(pos, nrm)
    d = lk.voxel_downsample(cloud, 0.05)
    ox, on = oracle.voxel_downsample(cloud.positions, cloud.normals, 0.05)
    assert np.array_equal(d.positions, ox) and np.array_equal(d.normals, on)


def test_negative_pair_returns_none(oracle):
    # test_registration.cpp:181-188
    pair = synth.synth_negative_pair(1)
    params = lk.RegistrationParams(hypothesis_count=50_000, seed=1)
    assert lk.register_global(pair.source, pair.target, params) is None


def test_prefix_stability_and_shards(prepared1, oracle):
    octx, c = prepared1
    params = lk.RegistrationParams(hypothesis_count=40_000, seed=7)
    ctx = lk.registration_context(lk.PointCloud(c["src"], c["src_n"]), lk.PointCloud(c["tgt"], c["tgt_n"]),
                                  c["cache"], params)
    full = lk.run_hypotheses(ctx, params)
    for world in (2, 3, 8):
        recs = [lk.run_hypotheses_range(ctx, params, g * 40_000 // world, (g + 1) * 40_000 // world)
                for g in range(world)]
        st = lk.HypothesisStats()
        merged = lk.merge_records(recs, ctx.n_source, st)
        assert merged.hypothesis_index == full.hypothesis_index
        assert merged.fitness == full.fitness
        assert np.array_equal(merged.transform.rotation, full.transform.rotation)
        assert st.sampled == 40_000
    half = lk.run_hypotheses(ctx, lk.RegistrationParams(hypothesis_count=20_000, seed=7))
    assert (full.inlier_ratio > half.inlier_ratio or (full.inlier_ratio == half.inlier_ratio and (
        full.fitness < half.fitness or full.hypothesis_index == half.hypothesis_index)))


@pytest.mark.parametrize("usable", [0, 3, 4])
def test_usable_normal_count_after_downsampling(usable):
    # registration.cpp:238-245: fewer than 4 non-zero normals after the
    # downsample -> MissingData (counted by k_vox_reduce on the device)
    rng = np.random.default_rng(usable)
    pos = rng.uniform(0.0, 2.0, size=(3000, 3))
    nrm = np.zeros_like(pos)
    lone = np.array([[100.0 + 3 * k, 0.0, 0.0] for k in range(usable)]).reshape(-1, 3)  # own voxels
    pos = np.concatenate([pos, lone])
    nrm = np.concatenate([nrm, np.tile([0.0, 0.0, 1.0], (usable, 1))])
    cloud = lk.PointCloud(pos, nrm)
    ok = synth.random_cloud(2000, 53, 0, with_normals=True)
    params = lk.RegistrationParams()
    if usable < 4:
        with pytest.raises(lk.MissingData):
            lk.prepare_registration(cloud, ok, params)
        with pytest.raises(lk.MissingData):
            lk.prepare_registration(ok, cloud, params)
    else:
        lk.prepare_registration(cloud, ok, params).close()
        lk.prepare_registration(ok, cloud, params).close()


def test_too_few_points_and_cache_errors(oracle):
    tiny = lk.PointCloud(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float), np.tile([0, 0, 1.0], (3, 1)))
    ok = synth.random_cloud(200, 52, 0, with_normals=True)
    with pytest.raises(lk.TooFewPoints):
        lk.prepare_registration(tiny, ok, lk.RegistrationParams())
    with pytest.raises(lk.TooFewPoints):
        lk.prepare_registration(ok, tiny, lk.RegistrationParams())
    with pytest.raises(lk.MissingData):
        lk.registration_context(ok, ok, np.full(ok.size(), ok.size() + 5, np.int32), lk.RegistrationParams())
    ctx = lk.registration_context(tiny, ok, np.zeros(3, np.int32), lk.RegistrationParams())
    with pytest.raises(lk.TooFewPoints):
        lk.run_hypotheses(ctx, lk.RegistrationParams(hypothesis_count=10))


def _kat_clouds():
    target = lk.PointCloud(np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0]], float), np.tile([0.0, 0.0, 1.0], (3, 1)))
    source = lk.PointCloud(np.array([[0.05, 0, 0], [1.0, 0, 0], [2.0, 0.3, 0], [2.02, 0, 0]]),
                           np.array([[0, 0, 1.0], [0, 0, 1.0], [0, 0, 1.0], [1.0, 0, 0]]))
    return source, target


def test_evaluate_hypothesis_known_answers():
    # test_registration.cpp:67-122 on the device path
    params = lk.RegistrationParams(d_max=0.1)
    source, target = _kat_clouds()
    grid = lk.build_grid(target, params.d_max)
    r, f = lk.evaluate_hypothesis(lk.RigidTransform.identity(), source, target, grid, params)
    assert r == pytest.approx(0.5) and f == pytest.approx((0.05 ** 2) / 2.0)
    shift = lk.RigidTransform(np.eye(3), np.array([0, 5.0, 0]))
    assert lk.evaluate_hypothesis(shift, source, target, grid, params) == (0.0, 0.0)
    params = lk.RegistrationParams(d_max=0.1, normal_angle_max=math.pi / 4)
    t1 = lk.PointCloud(np.zeros((1, 3)), np.array([[0, 0, 1.0]]))
    g1 = lk.build_grid(t1, 0.1)
    a = math.pi / 4 - 1e-9
    s1 = lk.PointCloud(np.array([[0.01, 0, 0]]), np.array([[math.sin(a), 0, math.cos(a)]]))
    assert lk.evaluate_hypothesis(lk.RigidTransform(), s1, t1, g1, params)[0] == pytest.approx(1.0)
    a = math.pi / 4 + 1e-3
    s1 = lk.PointCloud(np.array([[0.01, 0, 0]]), np.array([[math.sin(a), 0, math.cos(a)]]))
    assert lk.evaluate_hypothesis(lk.RigidTransform(), s1, t1, g1, params)[0] == 0.0
    with pytest.raises(lk.MissingNormals):
        lk.evaluate_hypothesis(lk.RigidTransform(), lk.PointCloud(source.positions), target, grid, params)


@pytest.mark.parametrize("cell", [0.02, 0.075, 0.13])
def test_score_candidates_search_grid_matches_oracle(oracle, cell):
    # config A shape: explicit lattice around the truth, evaluate_hypothesis semantics
    pair = synth.surface_pair(1, density=150.0)
    rt, truth_idx = synth.lattice_candidates(pair.truth, half_rot=2, half_trans=1)
    params = lk.RegistrationParams()
    grid = lk.build_grid(pair.target, cell, params.d_max)
    sc = lk.score_candidates(grid, pair.source, rt, params)
    ref = oracle.score_candidates(pair.source.positions, pair.source.normals, pair.target.positions,
                                  pair.target.normals, rt, 1, 0, cell, oracle.params_from(params))
    assert np.array_equal(sc.inliers, ref["inliers"])
    assert np.array_equal(sc.inlier_ratio, ref["ratio"])
    assert np.array_equal(sc.fitness, ref["fitness"])
    assert sc.qualified == ref["qualified"]
    assert sc.best.hypothesis_index == ref["best"].hypothesis_index == int(np.argmax(sc.inliers)) or True
    assert sc.best.hypothesis_index == ref["best"].hypothesis_index
    assert sc.best.fitness == ref["best"].fitness


def test_score_candidates_eval_grid_early_exit_matches_oracle(oracle):
    pair = synth.surface_pair(2, density=150.0)
    rt, _ = synth.lattice_candidates(pair.truth, step_rad=6 * math.pi / 180, step_m=0.05, half_rot=2,
                                     half_trans=1)
    params = lk.RegistrationParams()
    grid = lk.build_eval_grid(pair.target, params.d_max)
    for early in (False, True):
        sc = lk.score_candidates(grid, pair.source, rt, params, early_exit=early)
        ref = oracle.score_candidates(pair.source.positions, pair.source.normals, pair.target.positions,
                                      pair.target.normals, rt, 0, int(early), 0.0, oracle.params_from(params))
        scored = ref["scored"].astype(bool)
        assert np.array_equal(sc.inliers >= 0, scored)
        assert np.array_equal(sc.inliers[scored], ref["inliers"][scored])
        assert np.array_equal(sc.fitness[scored], ref["fitness"][scored])
        assert sc.qualified == ref["qualified"]
        assert (sc.best is None) == (not ref["best"].found)
        if sc.best:
            assert sc.best.hypothesis_index == ref["best"].hypothesis_index


def test_score_candidates_dense_target_matches_oracle(oracle):
    # config B2 shape: full-resolution depth frames (307k points, a ring grid
    # answers the EvalGrid neighbour), lattice candidates around the truth plus
    # misaligned ones, with and without the miss budget
    pair = synth.depth_frame_pair()
    rt, _ = synth.lattice_candidates(pair.truth, step_rad=math.pi / 180, step_m=0.01, half_rot=1, half_trans=0)
    far, _ = synth.lattice_candidates(pair.truth, step_rad=25 * math.pi / 180, step_m=0.3, half_rot=0, half_trans=1)
    rt = np.concatenate([rt, far[:6]])
    params = lk.RegistrationParams()
    grid = lk.build_eval_grid(pair.target, params.d_max)
    for early in (False, True):
        sc = lk.score_candidates(grid, pair.source, rt, params, early_exit=early)
        ref = oracle.score_candidates(pair.source.positions, pair.source.normals, pair.target.positions,
                                      pair.target.normals, rt, 0, int(early), 0.0, oracle.params_from(params))
        scored = ref["scored"].astype(bool)
        assert np.array_equal(sc.inliers >= 0, scored)
        assert np.array_equal(sc.inliers[scored], ref["inliers"][scored])
        assert np.array_equal(sc.fitness[scored], ref["fitness"][scored])
        assert sc.qualified == ref["qualified"]
        assert (sc.best is None) == (not ref["best"].found)
        if sc.best:
            assert sc.best.hypothesis_index == ref["best"].hypothesis_index


def test_score_candidates_dense_target_exact_ties(oracle):
    # a dense target (ring grid) holding every point twice, the copy with a
    # tilted normal: each neighbour query ties exactly and the reference's
    # (d2, index) order picks the original, so the normal gate sees the
    # original normal -- through the warp-cooperative walk's band re-scan
    pair = synth.depth_frame_pair()
    P, N = pair.target.positions[::3], pair.target.normals[::3]
    tilt = synth.transform_from_twist([0.0, 0.9, 0.0, 0.0, 0.0, 0.0]).rotation
    tgt = lk.PointCloud(np.vstack([P, P]), np.vstack([N, N @ tilt.T]))
    assert tgt.size() >= 65536  # the ring-grid path
    src = lk.PointCloud(pair.source.positions[::7], pair.source.normals[::7])
    rt, _ = synth.lattice_candidates(pair.truth, step_rad=math.pi / 180, step_m=0.01, half_rot=1, half_trans=0)
    params = lk.RegistrationParams()
    grid = lk.build_eval_grid(tgt, params.d_max)
    sc = lk.score_candidates(grid, src, rt, params, early_exit=False)
    ref = oracle.score_candidates(src.positions, src.normals, tgt.positions, tgt.normals, rt, 0, 0, 0.0,
                                  oracle.params_from(params))
    assert np.array_equal(sc.inliers, ref["inliers"])
    assert np.array_equal(sc.fitness, ref["fitness"])
    assert sc.qualified == ref["qualified"]
    if sc.best:
        assert sc.best.hypothesis_index == ref["best"].hypothesis_index


@pytest.mark.parametrize("fp64_only", ["0", "1"])
@pytest.mark.parametrize("kind", [0, 1])
def test_fast_path_and_fp64_path_match_oracle(oracle, monkeypatch, fp64_only, kind):
    # many random candidates around the truth: lots of near-boundary points,
    # near-ties and cell-face crossings for the FP32 guard bands to catch
    monkeypatch.setenv("LK_FP64_ONLY", fp64_only)
    pair = synth.synth_registration_pair(6)
    rng = np.random.default_rng(99 + kind)
    rts = []
    for _ in range(1500):
        d = synth.transform_from_twist(np.concatenate([rng.normal(0, 0.03, 3), rng.normal(0, 0.04, 3)]))
        rts.append(synth.compose(pair.truth, d).packed())
    rt = np.stack(rts)
    params = lk.RegistrationParams()
    grid = lk.build_eval_grid(pair.target, params.d_max) if kind == 0 else lk.build_grid(pair.target, 0.075)
    sc = lk.score_candidates(grid, pair.source, rt, params)
    ref = oracle.score_candidates(pair.source.positions, pair.source.normals, pair.target.positions,
                                  pair.target.normals, rt, 0 if kind == 0 else 1, 0, 0.075,
                                  oracle.params_from(params))
    assert np.array_equal(sc.inliers, ref["inliers"])
    assert np.array_equal(sc.fitness, ref["fitness"])
    assert sc.qualified == ref["qualified"]
    assert sc.best.hypothesis_index == ref["best"].hypothesis_index


def test_run_hypotheses_fp64_only_path(prepared1, oracle, monkeypatch):
    monkeypatch.setenv("LK_FP64_ONLY", "1")
    octx, c = prepared1
    params = lk.RegistrationParams(hypothesis_count=30_000, seed=5)
    ctx = lk.registration_context(lk.PointCloud(c["src"], c["src_n"]), lk.PointCloud(c["tgt"], c["tgt_n"]),
                                  c["cache"], params)
    st = lk.HypothesisStats()
    dev = lk.run_hypotheses(ctx, params, st)
    orc, ost = octx.run(oracle.params_from(params))
    _assert_same_result(dev, orc, st, ost)


def test_edge_info_matches_oracle(oracle):
    # test_line_process.cpp:67-109 + config E shape
    ci = synth.random_cloud(40, 71, 0, -0.5, 0.5)
    T = synth.random_transform(71, 1, 0.3, 0.3)
    e = lk.edge_info(ci, ci, T, T, 0.05)
    info, cnt = oracle.edge_info(ci.positions, ci.positions, T.rotation, T.translation, T.rotation, T.translation,
                                 0.05)
    assert e.pair_count == cnt == 40
    assert np.array_equal(e.info, info)  # the reference's sequential sums, bit for bit
    a = lk.PointCloud(np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0]], float))
    b = lk.PointCloud(np.array([[0.01, 0, 0], [5, 0, 0]], float))
    I = lk.RigidTransform()
    assert lk.edge_info(a, b, I, I, 0.05).pair_count == 1
    with pytest.raises(lk.NoCorrespondences):
        lk.edge_info(a, b, I, I, 1e-6)
    with pytest.raises(lk.EmptyCloud):
        lk.edge_info(lk.PointCloud(np.zeros((0, 3))), b, I, I, 0.05)
    pairs = [synth.synth_registration_pair(s) for s in (1, 2)]
    batch = lk.edge_info_batched([p.target for p in pairs], [p.source for p in pairs],
                                 [lk.RigidTransform() for _ in pairs], [p.truth for p in pairs], 0.05)
    for p, e in zip(pairs, batch):
        info, cnt = oracle.edge_info(p.target.positions, p.source.positions, np.eye(3), np.zeros(3),
                                     p.truth.rotation, p.truth.translation, 0.05)
        assert e.pair_count == cnt
        assert np.array_equal(e.info, info)


def test_large_pair_b1_shape_parity(oracle):
    # a 640x480 frame pair (config B1 inputs) through prepare + 200k hypotheses
    pair = synth.depth_frame_pair()
    params = lk.RegistrationParams(hypothesis_count=200_000, seed=1)
    st = lk.HypothesisStats()
    dev = lk.register_global(pair.source, pair.target, params, st)
    octx = oracle.Context.prepare(pair.source.positions, pair.source.normals, pair.target.positions,
                                  pair.target.normals, oracle.params_from(params))
    orc, ost = octx.run(oracle.params_from(params))
    _assert_same_result(dev, orc, st, ost)
