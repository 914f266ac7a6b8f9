"""Batched loop verification (config E; north-star item 5) against the oracle:
edge_info (line_process.cpp:11-33), the propose_loops overlap count
(fragments.cpp:67-100) and evaluate_hypothesis (registration.cpp:53-78) per
pair, all bit-exact (the device keeps the reference's sequential sums)."""
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


def _oracle_pair(oracle, Q, P, Ti, Tj, T, vp):
    info, cnt = (np.zeros((6, 6)), 0)
    try:
        info, cnt = oracle.edge_info(Q.positions, P.positions, Ti.rotation, Ti.translation, Tj.rotation,
                                     Tj.translation, vp.epsilon)
    except oracle.OracleError as e:
        assert e.code == 6
    hits = oracle.overlap_hits(P.positions, Tj.rotation, Tj.translation, Q.positions, Ti.rotation, Ti.translation,
                               vp.overlap_radius)
    op = oracle.params(d_max=vp.d_max, normal_angle_max=vp.normal_angle_max)
    ratio, fit, inl = oracle.evaluate_hypothesis(T.rotation, T.translation, P.positions, P.normals, Q.positions,
                                                 Q.normals, vp.grid_cell if vp.grid_cell > 0 else vp.d_max, op)
    return info, cnt, hits, ratio, fit, inl


@pytest.mark.parametrize("grid_cell", [0.0, 0.03])
def test_verify_batch_matches_oracle(oracle, grid_cell):
    pairs = [synth.synth_registration_pair(s) for s in range(1, 7)]
    Q = [p.target for p in pairs]
    P = [p.source for p in pairs]
    I = lk.RigidTransform()
    Ti = [I] * len(pairs)
    Tj = [p.truth for p in pairs]
    T = [p.truth for p in pairs]
    # a pair with a wrong measurement and a non-identity earlier pose
    Ti[2] = synth.random_transform(5, 3, 0.5, 0.5)
    Tj[2] = synth.compose(Ti[2], pairs[2].truth)
    T[4] = synth.compose(synth.transform_from_twist([0.2, 0.0, 0.1, 0.3, 0.0, 0.0]), pairs[4].truth)
    # far apart: no edge correspondences, no overlap
    Tj[5] = synth.compose(lk.RigidTransform(np.eye(3), np.array([50.0, 0, 0])), pairs[5].truth)
    vp = lk.VerifyParams(grid_cell=grid_cell)
    out = lk.verify_batch(Q, P, Ti, Tj, T, vp)
    for k in range(len(pairs)):
        info, cnt, hits, ratio, fit, inl = _oracle_pair(oracle, Q[k], P[k], Ti[k], Tj[k], T[k], vp)
        r = out[k]
        assert r.info.pair_count == cnt, k
        assert np.array_equal(r.info.info, info), k
        assert r.overlap_hits == hits, k
        assert r.overlap == hits / P[k].size()
        assert r.inliers == inl, k
        assert r.inlier_ratio == ratio, k
        assert r.fitness == fit, k
    assert out[5].info.pair_count == 0 and out[5].overlap_hits == 0
    assert out[0].overlap > 0.5 and out[0].inlier_ratio > 0.3


def test_verify_batch_errors():
    pair = synth.synth_registration_pair(1)
    I = lk.RigidTransform()
    with pytest.raises(lk.EmptyCloud):
        lk.verify_batch([lk.PointCloud(np.zeros((0, 3)), np.zeros((0, 3)))], [pair.source], [I], [I], [I])
    with pytest.raises(lk.MissingNormals):
        lk.verify_batch([lk.PointCloud(pair.target.positions)], [pair.source], [I], [I], [I])
    assert lk.verify_batch([], [], [], [], []) == []


def test_verified_loops_weighted_by_the_line_process():
    """Row a11 on top of the batch: the truth measurement of a pair is kept
    (residual 0, weight 1), a measurement off by 0.5 rad / 0.6 m is rejected."""
    pairs = [synth.synth_registration_pair(s) for s in (2, 3)]
    Q = [p.target for p in pairs]
    P = [p.source for p in pairs]
    I = [lk.RigidTransform()] * 2
    Tj = [p.truth for p in pairs]
    out = lk.verify_batch(Q, P, I, Tj, Tj, lk.VerifyParams())
    off = synth.compose(synth.transform_from_twist([0.5, 0.0, 0.0, 0.6, 0.0, 0.0]), pairs[1].truth)
    # consistent measurement: rel = T_i^-1 T_j (residual rel T_j^-1 T_i = identity)
    rel = [synth.compose(synth.inverse(I[0]), Tj[0]), synth.compose(off, synth.compose(synth.inverse(Tj[1]), Tj[1]))]
    w, acc = lk.loop_weights(I, Tj, rel, [o.info for o in out])
    assert out[0].info.pair_count > 0 and out[1].info.pair_count > 0
    assert w[0] == pytest.approx(1.0, abs=1e-9) and acc[0]
    assert w[1] < 0.25 and not acc[1]


def test_verify_batch_large_batch_equals_small_batches(oracle):
    """A 70-pair batch from page-locked clouds (the zero-copy gather path)
    equals the same pairs verified in batches of 8, and a few are checked
    against the oracle. torch is imported after the library: the library
    must not have pulled a second NCCL into the process."""
    import torch
    pairs = [synth.synth_registration_pair(s) for s in range(1, 71)]
    keep = []

    def pin(c):  # page-locked clouds: the zero-copy gather path of the bench
        tp = torch.from_numpy(np.ascontiguousarray(c.positions)).pin_memory()
        tn = torch.from_numpy(np.ascontiguousarray(c.normals)).pin_memory()
        keep.extend([tp, tn])
        return lk.PointCloud(tp.numpy(), tn.numpy())

    Q = [pin(p.target) for p in pairs]
    P = [pin(p.source) for p in pairs]
    Ti = [lk.RigidTransform() for _ in pairs]
    Tj = [p.truth for p in pairs]
    T = [p.truth if k % 5 else synth.compose(synth.transform_from_twist([0.1, 0, 0, 0.1, 0, 0]), p.truth)
         for k, p in enumerate(pairs)]
    vp = lk.VerifyParams()
    big = lk.verify_batch(Q, P, Ti, Tj, T, vp)
    for a in range(0, len(pairs), 8):
        small = lk.verify_batch(Q[a:a + 8], P[a:a + 8], Ti[a:a + 8], Tj[a:a + 8], T[a:a + 8], vp)
        for k, r in enumerate(small):
            b = big[a + k]
            assert b.info.pair_count == r.info.pair_count and np.array_equal(b.info.info, r.info.info), a + k
            assert b.overlap_hits == r.overlap_hits and b.inliers == r.inliers and b.fitness == r.fitness, a + k
    for k in (0, 17, 35, 69):
        info, cnt, hits, ratio, fit, inl = _oracle_pair(oracle, Q[k], P[k], Ti[k], Tj[k], T[k], vp)
        r = big[k]
        assert r.info.pair_count == cnt and np.array_equal(r.info.info, info), k
        assert r.overlap_hits == hits and r.inliers == inl and r.fitness == fit, k
