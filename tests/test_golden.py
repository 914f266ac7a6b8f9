"""Committed golden vectors (tests/golden/golden.json, made by
tests/golden/make_golden.py from the KAT-pinned oracle): the oracle must keep
reproducing them (CPU) and the B200 path must equal them (GPU)."""
import json
import os

import numpy as np
import pytest

from paper_1801_01572_b200 import synth

G = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.json")))


def unhex(v):
    return np.array([float.fromhex(x) for x in v])


def test_oracle_rng_golden(oracle):
    for key, vals in G["rng_u64"].items():
        s, k = map(int, key.split(","))
        assert oracle.rng_u64(s, k, 8).tolist() == vals
    for key, vals in G["rng_bounded"].items():
        s, k, b = map(int, key.split(","))
        assert oracle.rng_bounded(s, k, b, 16).tolist() == vals


def test_oracle_kabsch_golden(oracle):
    for case in G["kabsch"]:
        R, t = oracle.kabsch(unhex(case["src"]).reshape(4, 3), unhex(case["dst"]).reshape(4, 3))
        assert np.array_equal(R.reshape(-1), unhex(case["R"]))
        assert np.array_equal(t, unhex(case["t"]))


def test_fixture_generators_golden():
    for r in G["run_hypotheses"][::2]:
        pair = synth.synth_registration_pair(r["pair"])
        assert pair.source.size() == r["n_src"] and pair.target.size() == r["n_tgt"]
        assert float(pair.source.positions.sum()).hex() == r["src_sum"]
        assert float(pair.target.positions.sum()).hex() == r["tgt_sum"]


@pytest.mark.slow
def test_oracle_run_hypotheses_golden(oracle):
    for r in G["run_hypotheses"]:
        pair = synth.synth_registration_pair(r["pair"])
        p = oracle.params(hypothesis_count=r["H"], seed=r["seed"])
        ctx = oracle.Context.prepare(pair.source.positions, pair.source.normals, pair.target.positions,
                                     pair.target.normals, p)
        res, st = ctx.run(p)
        assert res.hypothesis_index == r["index"] and res.inliers == r["inliers"]
        assert float(res.fitness).hex() == r["fitness"]
        assert np.array_equal(res.R.reshape(-1), unhex(r["R"]))
        assert {k: st[k] for k in r["stats"]} == r["stats"]


@pytest.mark.gpu
def test_device_run_hypotheses_golden():
    import paper_1801_01572_b200 as lk
    for r in G["run_hypotheses"]:
        pair = synth.synth_registration_pair(r["pair"])
        params = lk.RegistrationParams(hypothesis_count=r["H"], seed=r["seed"])
        st = lk.HypothesisStats()
        res = lk.register_global(pair.source, pair.target, params, st)
        assert (res is not None) == r["found"]
        assert res.hypothesis_index == r["index"] and res.inliers == r["inliers"]
        assert float(res.fitness).hex() == r["fitness"]
        assert np.array_equal(res.transform.rotation.reshape(-1), unhex(r["R"]))
        assert np.array_equal(res.transform.translation, unhex(r["t"]))
        assert {k: getattr(st, k) for k in r["stats"]} == r["stats"]


@pytest.mark.gpu
def test_device_score_candidates_golden():
    import paper_1801_01572_b200 as lk
    s = G["score_candidates"]
    pair = synth.surface_pair(s["seed"], density=s["density"])
    rt, truth_idx = synth.lattice_candidates(pair.truth, half_rot=s["half_rot"], half_trans=s["half_trans"])
    assert truth_idx == s["truth_index"]
    grid = lk.build_grid(pair.target, 0.075)
    sc = lk.score_candidates(grid, pair.source, rt, lk.RegistrationParams())
    assert sc.inliers.tolist() == s["inliers"]
    assert np.array_equal(sc.fitness, unhex(s["fitness"]))
    assert sc.best.hypothesis_index == s["best"] and sc.qualified == s["qualified"]


@pytest.mark.gpu
def test_device_edge_info_golden():
    import paper_1801_01572_b200 as lk
    e = G["edge_info"]
    pair = synth.synth_registration_pair(e["pair"])
    got = lk.edge_info(pair.target, pair.source, lk.RigidTransform(), pair.truth, e["eps"])
    ref = np.array(e["info"]).reshape(6, 6)
    assert got.pair_count == e["pair_count"]
    assert np.abs(got.info - ref).max() <= 1e-9 * np.abs(ref).max()
