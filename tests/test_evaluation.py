"""Registration logs and Table-I scoring (paper_1801_01572_b200/evaluation.py and
`loopkit_b200 evaluate --mode registration`): the reference's .log format
(proj/src/io.cpp:341-381) and eval_registration (proj/src/metrics.cpp:112-156),
checked on the reference's own test cases (proj/tests/test_metrics.cpp:155-209)
and on the scoring of real B200 registration runs."""
import math
import subprocess

import numpy as np
import pytest

import paper_1801_01572_b200 as lk
from paper_1801_01572_b200 import synth

from test_cli import CLI, write_ply


def _entry(i, j, n, T):
    return lk.log_entry(i, j, n, T.rotation, T.translation)


def _shift(T, dx):
    return lk.RigidTransform(T.rotation.copy(), T.translation + np.array([dx, 0.0, 0.0]))


def _rot_z(a):
    c, s = math.cos(a), math.sin(a)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def _case_one():
    # test_metrics.cpp:155-188: three truth pairs; one near result (0.05 m off),
    # one far (1 m off), one pair absent from the truth.
    t01 = synth.random_transform(43, 0, 1.0, 1.0)
    t02 = synth.random_transform(43, 1, 1.0, 1.0)
    t13 = synth.random_transform(43, 2, 1.0, 1.0)
    truth = [_entry(1, 0, 4, t01), _entry(2, 0, 4, t02), _entry(3, 1, 4, t13)]
    results = [_entry(1, 0, 4, _shift(t01, 0.05)), _entry(2, 0, 4, _shift(t02, 1.0)), _entry(2, 1, 4, t13)]
    duped = [_entry(1, 0, 4, t01), _entry(1, 0, 4, t01)]
    return truth, results, duped


def test_eval_registration_reference_case():
    truth, results, duped = _case_one()
    s = lk.eval_registration(results, truth)
    assert (s.correct, s.truth_count, s.result_count) == (1, 3, 3)
    assert s.recall == pytest.approx(1 / 3) and s.precision == pytest.approx(1 / 3)
    s = lk.eval_registration(duped, truth)  # credited once; precision pays
    assert s.correct == 1 and s.recall == pytest.approx(1 / 3) and s.precision == pytest.approx(0.5)
    s = lk.eval_registration([], truth)
    assert (s.recall, s.precision, s.correct, s.result_count) == (0.0, 0.0, 0, 0)
    s = lk.eval_registration(results, [])
    assert (s.recall, s.precision, s.correct, s.truth_count, s.result_count) == (0.0, 0.0, 0, 0, 3)


def test_eval_registration_probe_lever_arm():
    # test_metrics.cpp:190-209: 0.01 rad is harmless on the unit cube, fatal at 40 m
    gt = lk.log_entry(2, 0, 3, np.eye(3), np.zeros(3))
    est = lk.log_entry(2, 0, 3, _rot_z(0.01), np.zeros(3))
    assert lk.eval_registration([est], [gt]).correct == 1
    probes = [np.array([[40.0, 0.1 * i, 0.0] for i in range(16)])]
    assert lk.eval_registration([est], [gt], probes).correct == 0
    # an empty probe cloud falls back to the cube; j outside the probes too
    assert lk.eval_registration([est], [gt], [np.zeros((0, 3))]).correct == 1
    assert lk.eval_registration([lk.log_entry(2, 5, 3, _rot_z(0.01), np.zeros(3))],
                                [lk.log_entry(2, 5, 3, np.eye(3), np.zeros(3))], probes).correct == 1
    # the bound is strict (0.25 m is exact on the cube corners)
    near = lk.log_entry(2, 0, 3, np.eye(3), np.array([0.25, 0.0, 0.0]))
    assert lk.eval_registration([near], [gt], rmse_max=0.25).correct == 0
    assert lk.eval_registration([near], [gt], rmse_max=0.2500001).correct == 1


def test_registration_log_round_trip_and_errors(tmp_path):
    truth, results, _ = _case_one()
    p = tmp_path / "a.log"
    lk.write_registration_log(str(p), truth)
    back = lk.read_registration_log(str(p))
    assert [(e.i, e.j, e.n) for e in back] == [(e.i, e.j, e.n) for e in truth]
    for a, b in zip(back, truth):
        assert np.array_equal(a.transform, b.transform)  # %.17g round-trips doubles
    # comments, blank lines and CRLF are accepted
    text = p.read_text()
    q = tmp_path / "b.log"
    q.write_text("# header\n\n" + text.replace("\n", "\r\n") + "  \n")
    assert len(lk.read_registration_log(str(q))) == 3
    bad = tmp_path / "bad.log"
    bad.write_text("1 0\n")
    with pytest.raises(lk.ParseError, match=r"bad.log:1: expected header line"):
        lk.read_registration_log(str(bad))
    bad.write_text("1 0 4\n1 0 0 0\n0 1 0\n")
    with pytest.raises(lk.ParseError, match=r"bad.log:3: expected 4 matrix values"):
        lk.read_registration_log(str(bad))
    bad.write_text("1 0 4\n1 0 0 0\n")
    with pytest.raises(lk.ParseError, match=r"truncated matrix block"):
        lk.read_registration_log(str(bad))


def _cli_eval(est, truth, frags=None, rmse_max=None):
    args = [CLI, "evaluate", "--mode", "registration", "--est", str(est), "--truth", str(truth)]
    if frags is not None:
        args += ["--frags", str(frags)]
    if rmse_max is not None:
        args += ["--rmse-max", repr(rmse_max)]
    r = subprocess.run(args, capture_output=True, text=True, timeout=60)
    return r


def _parse(out):
    kv = dict(line.split() for line in out.strip().splitlines())
    return float(kv["recall"]), float(kv["precision"]), int(kv["correct"])


def test_cli_evaluate_matches_python(tmp_path):
    truth, results, duped = _case_one()
    tp, rp, dp = tmp_path / "t.log", tmp_path / "r.log", tmp_path / "d.log"
    lk.write_registration_log(str(tp), truth)
    lk.write_registration_log(str(rp), results)
    lk.write_registration_log(str(dp), duped)
    for est in (rp, dp):
        r = _cli_eval(est, tp)
        assert r.returncode == 0, r.stderr
        s = lk.eval_registration(lk.read_registration_log(str(est)), truth)
        assert _parse(r.stdout) == (s.recall, s.precision, s.correct)
        assert r.stdout == "recall %.17g\nprecision %.17g\ncorrect %d\n" % (s.recall, s.precision, s.correct)
    # probes from --frags: fragment_0000.ply on a 40 m lever arm
    frags = tmp_path / "frags"
    frags.mkdir()
    probe, _ = write_ply(frags / "fragment_0000.ply", [[40.0, 0.1 * i, 0.0] for i in range(16)])
    gt = [lk.log_entry(2, 0, 3, np.eye(3), np.zeros(3))]
    est = [lk.log_entry(2, 0, 3, _rot_z(0.01), np.zeros(3))]
    lk.write_registration_log(str(tp), gt)
    lk.write_registration_log(str(rp), est)
    assert _parse(_cli_eval(rp, tp).stdout)[2] == 1
    assert _parse(_cli_eval(rp, tp, frags).stdout)[2] == 0
    assert _parse(_cli_eval(rp, tp, frags, rmse_max=1.0).stdout)[2] == 1
    assert lk.eval_registration(est, gt, [probe]).correct == 0
    # random logs: many pairs, duplicates, near-threshold errors
    rng = np.random.default_rng(7)
    truth, results = [], []
    for k in range(60):
        i, j = int(rng.integers(0, 8)), int(rng.integers(0, 8))
        T = synth.random_transform(100 + k, 0, 1.0, 2.0)
        truth.append(_entry(i, j, 8, T))
        for _ in range(int(rng.integers(0, 3))):
            results.append(_entry(i, j, 8, _shift(T, float(rng.uniform(0.0, 0.4)))))
    rng.shuffle(results)
    lk.write_registration_log(str(tp), truth)
    lk.write_registration_log(str(rp), results)
    s = lk.eval_registration(lk.read_registration_log(str(rp)), lk.read_registration_log(str(tp)))
    assert 0 < s.correct < len(truth)
    assert _parse(_cli_eval(rp, tp).stdout) == (s.recall, s.precision, s.correct)
    # errors: unknown mode, missing frags dir, malformed log
    assert "error:" in subprocess.run([CLI, "evaluate", "--mode", "ate", "--est", str(rp), "--truth", str(tp)],
                                      capture_output=True, text=True).stderr
    r = _cli_eval(rp, tp, tmp_path / "nowhere")
    assert r.returncode == 1 and "no fragment_%04d.ply files" in r.stderr
    (tmp_path / "bad.log").write_text("1 0\n")
    r = _cli_eval(tmp_path / "bad.log", tp)
    assert r.returncode == 1 and "bad.log:1: expected header line" in r.stderr


@pytest.mark.gpu
def test_table1_scoring_of_b200_registrations(tmp_path):
    """Register fragment pairs on the B200 path, write the log and score it
    against the truth log the way the reference scores its runs (Table I)."""
    if lk.device_count() == 0:
        pytest.fail("no CUDA device visible: -m gpu tests must run on the B200 box")
    params = lk.RegistrationParams(hypothesis_count=200_000, seed=3)
    truth, results = [], []
    for k in range(4):
        pair = synth.synth_registration_pair(k + 1)
        truth.append(_entry(k + 1, 0, 6, pair.truth))
        r = lk.register_global(pair.source, pair.target, params)
        assert r is not None
        results.append(_entry(k + 1, 0, 6, r.transform))
    neg = synth.synth_negative_pair(9)
    r = lk.register_global(neg.source, neg.target, params)
    if r is not None:  # a false positive costs precision, never recall
        results.append(_entry(5, 0, 6, r.transform))
    tp, rp = tmp_path / "truth.log", tmp_path / "est.log"
    lk.write_registration_log(str(tp), truth)
    lk.write_registration_log(str(rp), results)
    s = lk.eval_registration(lk.read_registration_log(str(rp)), lk.read_registration_log(str(tp)))
    assert s.correct == 4 and s.recall == 1.0
    assert s.precision == 4 / len(results)
    assert _parse(_cli_eval(rp, tp).stdout) == (s.recall, s.precision, s.correct)
