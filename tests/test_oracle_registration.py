"""Oracle pins: scoring, selection and end-to-end properties
(proj/tests/test_registration.cpp:67-198, test_line_process.cpp:67-109,
SPEC.md invariants), plus EvalGrid/evaluate_against_grid consistency."""
import math

import numpy as np
import pytest

from paper_1801_01572_b200 import synth


def _kat_clouds():
    target = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0]], float)
    tn = np.tile([0.0, 0.0, 1.0], (3, 1))
    source = np.array([[0.05, 0, 0], [1.0, 0, 0], [2.0, 0.3, 0], [2.02, 0, 0]])
    sn = np.array([[0, 0, 1.0], [0, 0, 1.0], [0, 0, 1.0], [1.0, 0, 0]])
    return source, sn, target, tn


def test_evaluate_hypothesis_known_answer(oracle):
    # test_registration.cpp:67-97
    s, sn, t, tn = _kat_clouds()
    p = oracle.params(d_max=0.1)
    r, f, inl = oracle.evaluate_hypothesis(np.eye(3), np.zeros(3), s, sn, t, tn, 0.1, p)
    assert r == pytest.approx(0.5)
    assert f == pytest.approx((0.05 ** 2 + 0.0) / 2.0)
    assert inl == 2
    r2, f2, _ = oracle.evaluate_hypothesis(np.eye(3), np.array([0, 5.0, 0]), s, sn, t, tn, 0.1, p)
    assert r2 == 0.0 and f2 == 0.0


def test_normal_gate_inclusive(oracle):
    # test_registration.cpp:99-122
    p = oracle.params(d_max=0.1, normal_angle_max=math.pi / 4)
    t, tn = np.zeros((1, 3)), np.array([[0, 0, 1.0]])
    s = np.array([[0.01, 0, 0]])
    a = math.pi / 4 - 1e-9
    r, _, _ = oracle.evaluate_hypothesis(np.eye(3), np.zeros(3), s, np.array([[math.sin(a), 0, math.cos(a)]]), t, tn,
                                         0.1, p)
    assert r == pytest.approx(1.0)
    a = math.pi / 4 + 1e-3
    r, _, _ = oracle.evaluate_hypothesis(np.eye(3), np.zeros(3), s, np.array([[math.sin(a), 0, math.cos(a)]]), t, tn,
                                         0.1, p)
    assert r == 0.0


def test_spec_evaluate_examples(oracle):
    # SPEC.md:298-306 (P == Q, T = I -> 1.0 / 0; displaced 0.2 m -> 0; half overlap -> 0.5)
    c = synth.random_cloud(500, 31, 0, with_normals=True)
    p = oracle.params()
    r, f, _ = oracle.evaluate_hypothesis(np.eye(3), np.zeros(3), c.positions, c.normals, c.positions, c.normals,
                                         0.075, p)
    assert r == 1.0 and abs(f) < 1e-12
    r, _, _ = oracle.evaluate_hypothesis(np.eye(3), np.array([0.2, 0, 0]), c.positions, c.normals,
                                         c.positions + np.array([0.0, 0, 0]), c.normals, 0.075, p)
    assert r < 1.0
    half = c.positions.copy()
    far = c.positions[250:] + np.array([10.0, 0, 0])
    src = np.vstack([half[:250], far])
    r, f, _ = oracle.evaluate_hypothesis(np.eye(3), np.zeros(3), src, c.normals, c.positions, c.normals, 0.075, p)
    assert r == 0.5 and f == 0.0


def test_eval_grid_matches_evaluate_hypothesis(oracle):
    # registration.cpp:152-153: "Identical to evaluate_hypothesis for every
    # hypothesis it fully scores" (integer outcomes; fitness rounds differently)
    pair = synth.synth_registration_pair(2)
    s, t = pair.source, pair.target
    p = oracle.params()
    eg = oracle.EvalGrid(t.positions, t.normals, p.d_max)
    cos_max = math.cos(p.normal_angle_max)
    for k in range(6):
        d = synth.transform_from_twist([0.01 * k, -0.02 * k, 0.015 * k, 0.01 * k, 0, -0.01 * k])
        T = synth.compose(pair.truth, d)
        ok, r, f, inl, vis = eg.evaluate(s.positions, s.normals, T.rotation, T.translation, p.d_max, cos_max,
                                         10**12)
        r2, f2, inl2 = oracle.evaluate_hypothesis(T.rotation, T.translation, s.positions, s.normals, t.positions,
                                                  t.normals, p.d_max, p)
        assert ok and inl == inl2 and vis == s.size()
        assert f == pytest.approx(f2, rel=1e-12)


def test_eval_grid_layout(oracle):
    pair = synth.synth_registration_pair(2)
    t = pair.target
    eg = oracle.EvalGrid(t.positions, t.normals, 0.075)
    a = eg.arrays()
    lo = t.positions.min(0)
    assert np.array_equal(eg.origin, lo - 0.075)
    assert a["start"][0] == 0 and a["start"][-1] == t.size()
    # ascending original index inside every cell
    for c in np.nonzero(np.diff(a["start"]))[0][:500]:
        seg = a["index"][a["start"][c]:a["start"][c + 1]]
        assert (np.diff(seg) > 0).all()
    assert np.array_equal(a["slot_position"], t.positions[a["index"]])


@pytest.mark.slow
def test_run_hypotheses_deterministic_and_prefix_stable(oracle):
    # test_registration.cpp:124-160
    pair = synth.synth_registration_pair(3)
    p = oracle.params(hypothesis_count=20_000, seed=7, threads=1)
    ctx = oracle.Context.prepare(pair.source.positions, pair.source.normals, pair.target.positions,
                                 pair.target.normals, p)
    serial, st1 = ctx.run(p)
    assert serial.found
    for threads in (2, 4):
        p.threads = threads
        other, st = ctx.run(p)
        assert other.hypothesis_index == serial.hypothesis_index
        assert other.inlier_ratio == serial.inlier_ratio and other.fitness == serial.fitness
        assert np.array_equal(other.R, serial.R) and np.array_equal(other.t, serial.t)
        for k in ("prerejected", "degenerate", "evaluated", "qualified", "w_ref"):
            assert st[k] == st1[k]
    assert serial.hypothesis_index < 20_000
    p.threads = 0
    p.hypothesis_count = 40_000
    ext, _ = ctx.run(p)
    assert ext.found
    assert (ext.inlier_ratio > serial.inlier_ratio
            or (ext.inlier_ratio == serial.inlier_ratio and ext.fitness < serial.fitness)
            or (ext.inlier_ratio == serial.inlier_ratio and ext.fitness == serial.fitness
                and ext.hypothesis_index == serial.hypothesis_index))


@pytest.mark.slow
def test_register_global_recovers_planted_transform(oracle):
    # test_registration.cpp:162-179
    pair = synth.synth_registration_pair(1)
    p = oracle.params(hypothesis_count=100_000, seed=1)
    ctx = oracle.Context.prepare(pair.source.positions, pair.source.normals, pair.target.positions,
                                 pair.target.normals, p)
    r, st = ctx.run(p)
    assert r.found
    assert st["sampled"] == 100_000
    assert st["prerejected"] + st["degenerate"] + st["evaluated"] == st["sampled"]
    Rerr = pair.truth.rotation.T @ r.R
    ang = math.acos(max(-1.0, min(1.0, (np.trace(Rerr) - 1) / 2)))
    terr = np.linalg.norm(pair.truth.rotation.T @ (r.t - pair.truth.translation))
    assert ang < 3 * math.pi / 180
    assert terr < 0.05
    assert r.inlier_ratio >= 0.25 and r.fitness <= 0.075 ** 2 / 2


@pytest.mark.slow
def test_register_global_negative_pair(oracle):
    # test_registration.cpp:181-188
    pair = synth.synth_negative_pair(1)
    p = oracle.params(hypothesis_count=50_000, seed=1)
    ctx = oracle.Context.prepare(pair.source.positions, pair.source.normals, pair.target.positions,
                                 pair.target.normals, p)
    r, _ = ctx.run(p)
    assert not r.found


def test_prepare_rejects_unusable_inputs(oracle):
    # test_registration.cpp:190-198
    tiny = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float)
    ok = synth.random_cloud(200, 52, 0, with_normals=True)
    p = oracle.params()
    with pytest.raises(oracle.OracleError) as e:
        oracle.Context.prepare(tiny, np.tile([0, 0, 1.0], (3, 1)), ok.positions, ok.normals, p)
    assert e.value.code == 3
    with pytest.raises(oracle.OracleError) as e:
        oracle.Context.prepare(ok.positions, ok.normals, tiny, np.tile([0, 0, 1.0], (3, 1)), p)
    assert e.value.code == 3


def test_edge_info_known_answers(oracle):
    # test_line_process.cpp:67-109
    ci = synth.random_cloud(40, 71, 0, -0.5, 0.5).positions
    T = synth.random_transform(71, 1, 0.3, 0.3)
    info, cnt = oracle.edge_info(ci, ci, T.rotation, T.translation, T.rotation, T.translation, 0.05)
    assert cnt == 40
    expect = np.zeros((6, 6))
    for p in ci:
        S = np.array([[0, -p[2], p[1]], [p[2], 0, -p[0]], [-p[1], p[0], 0]])
        G = np.hstack([-S, np.eye(3)])
        expect += G.T @ G
    assert np.abs(info - expect).max() < 1e-9
    assert np.abs(info - info.T).max() < 1e-12
    assert np.linalg.eigvalsh(info).min() > -1e-9
    a = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0]], float)
    b = np.array([[0.01, 0, 0], [5, 0, 0]], float)
    I, z = np.eye(3), np.zeros(3)
    _, cnt = oracle.edge_info(a, b, I, z, I, z, 0.05)
    assert cnt == 1
    with pytest.raises(oracle.OracleError) as e:
        oracle.edge_info(a, b, I, z, I, z, 1e-6)
    assert e.value.code == 6
    with pytest.raises(oracle.OracleError) as e:
        oracle.edge_info(np.zeros((0, 3)), b, I, z, I, z, 0.05)
    assert e.value.code == 2


def test_voxel_downsample_first_index_order(oracle):
    # preprocess.cpp:14-59: one point per voxel, ordered by first input index
    rng = np.random.default_rng(5)
    pts = rng.uniform(-1, 1, size=(2000, 3))
    nrm = rng.normal(size=(2000, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    nrm[::7] = 0.0
    out, outn = oracle.voxel_downsample(pts, nrm, 0.2)
    keys = np.floor(pts / 0.2).astype(np.int64)
    _, first = np.unique(keys, axis=0, return_index=True)
    assert out.shape[0] == first.size
    order = np.sort(first)
    for k, i in enumerate(order[:50]):
        members = (keys == keys[i]).all(1)
        assert np.allclose(out[k], pts[members].mean(0), rtol=0, atol=1e-15)
        ns = nrm[members].sum(0)
        if np.linalg.norm(ns) > 1e-12:
            assert np.allclose(outn[k], ns / np.linalg.norm(ns), atol=1e-15)
