"""lk_propose_loops (include/loopkit_b200.h) on the device against the
reference's own outputs and its tests.

Ports proj/tests/test_fragments.cpp:150-200 ("propose_loops matches the
brute-force oracle", "never pairs adjacent fragments") with the same seeded
draws, and checks the reference golden case (tests/golden/ref_golden.json,
made by oracle/_ref's propose_loops) bit for bit. The overlap of every
proposal is also checked bitwise against the oracle's per-pair hit count
(or_overlap_hits, the fragments.cpp:93-99 loop restated).
"""
import json
import os

import numpy as np
import pytest

import paper_1801_01572_b200 as lk
from paper_1801_01572_b200 import synth

pytestmark = pytest.mark.gpu

G = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_golden.json")))


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if lk.device_count() == 0:
        pytest.fail("no CUDA device visible: -m gpu tests must run on the B200 box")


class Draws:
    """RngStream(seed, stream) consumed in order (proj/include/loopkit/rng.hpp),
    with GCC's right-to-left evaluation of Vec3(a(), b(), c()) arguments."""

    def __init__(self, oracle, seed, stream, n=1 << 16):
        self.u = oracle.rng_u64(seed, stream, n)
        self.k = 0

    def double(self, lo, hi):
        x = float(int(self.u[self.k]) >> 11) * 2.0 ** -53
        self.k += 1
        return lo + (hi - lo) * x

    def vec3(self, lo, hi):
        z = self.double(lo, hi)
        y = self.double(lo, hi)
        x = self.double(lo, hi)
        return np.array([x, y, z])


def _brute(frags, poses, loops, r, min_overlap):
    """test_fragments.cpp:113-146 propose_oracle: brute force with |p - q| <= r."""
    posed = [c @ T.rotation.T + T.translation for c, T in zip(frags, poses)]
    out = []
    n = len(frags)
    for i in range(2, n):
        for j in range(0, i - 1):
            if (i, j) in loops or (j, i) in loops:
                continue
            d = np.sqrt(((posed[i][:, None, :] - posed[j][None, :, :]) ** 2).sum(-1)).min(axis=1)
            ov = float((d <= r).sum()) / posed[i].shape[0]
            if ov >= min_overlap:
                out.append((i, j, ov))
    out.sort(key=lambda x: (-x[2], x[0], x[1]))
    return out


def test_propose_loops_matches_brute_force_oracle(oracle):
    """test_fragments.cpp:150-181: RngStream(65, 0), 4 trials of 6 fragments of
    60 points in [-0.4, 0.4]^3 at translations in [-0.5, 0.5]^3; odd trials add
    a loop edge (0, 3) that must suppress the pair (3, 0)."""
    rng = Draws(oracle, 65, 0)
    for trial in range(4):
        frags, poses = [], []
        for _ in range(6):
            frags.append(np.array([rng.vec3(-0.4, 0.4) for _ in range(60)]))
            poses.append(lk.RigidTransform(translation=rng.vec3(-0.5, 0.5)))
        loops = [(0, 3)] if trial % 2 == 1 else []
        got = lk.propose_loops([lk.PointCloud(f) for f in frags], poses, loops,
                               lk.LoopParams(overlap_radius=0.15, min_overlap=0.1))
        want = _brute(frags, poses, set(loops), 0.15, 0.1)
        assert [(p.i, p.j) for p in got] == [(i, j) for i, j, _ in want]
        for p, (_, _, ov) in zip(got, want):
            assert abs(p.overlap - ov) <= 1e-12 * max(1.0, ov)
            assert p.i >= p.j + 2
            hits = oracle.overlap_hits(frags[p.i], poses[p.i].rotation, poses[p.i].translation, frags[p.j],
                                       poses[p.j].rotation, poses[p.j].translation, 0.15)
            assert p.overlap == hits / frags[p.i].shape[0]
        if trial % 2 == 1:
            assert all((p.i, p.j) != (3, 0) for p in got)


def test_propose_loops_never_pairs_adjacent_fragments(oracle):
    """test_fragments.cpp:183-200: identical clouds and poses, min_overlap 0 ->
    only (2, 0)."""
    rng = Draws(oracle, 66, 0)
    shared = np.array([rng.vec3(-0.3, 0.3) for _ in range(50)])
    frags = [lk.PointCloud(shared.copy()) for _ in range(3)]
    poses = [lk.RigidTransform() for _ in range(3)]
    got = lk.propose_loops(frags, poses, [], lk.LoopParams(min_overlap=0.0))
    assert len(got) == 1 and (got[0].i, got[0].j) == (2, 0) and got[0].overlap > 0.9


def test_propose_loops_matches_reference_golden():
    g = G["propose_loops"]
    frags = [synth.random_cloud(n, s, 0, -0.4, 0.4) for s, n in g["clouds"]]
    poses = [synth.random_transform(s, 0, a, tr) for s, a, tr in g["poses"]]
    got = lk.propose_loops(frags, poses, [tuple(x) for x in g["loops"]],
                           lk.LoopParams(overlap_radius=g["overlap_radius"], min_overlap=g["min_overlap"]))
    assert [(p.i, p.j, float(p.overlap).hex()) for p in got] == [tuple(x) for x in g["proposals"]]


def test_propose_loops_errors():
    frags = [lk.PointCloud(np.zeros((3, 3))) for _ in range(3)]
    with pytest.raises(lk.MissingData):
        lk.propose_loops(frags, [lk.RigidTransform()] * 2)
    frags[1] = lk.PointCloud(np.zeros((0, 3)))
    with pytest.raises(lk.EmptyCloud):
        lk.propose_loops(frags, [lk.RigidTransform()] * 3)
    assert lk.propose_loops([], []) == []
