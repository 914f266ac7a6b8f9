"""Oracle pins: RNG (proj/include/loopkit/rng.hpp) and quadruple sampling /
pre-rejection (proj/tests/test_registration.cpp:16-65)."""
import math

import numpy as np


def test_splitmix64_published_vector(oracle):
    # SplitMix64 (Steele/Lea/Flood; Vigna's splitmix64.c) seeded with 0 yields
    # 0xE220A8397B1DCDAF first: splitmix64(0) is that output.
    assert oracle.lib().or_splitmix64(0) == 0xE220A8397B1DCDAF
    assert oracle.lib().or_splitmix64(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4


def test_rng_streams_are_pure_functions(oracle):
    a = oracle.rng_u64(99, 5, 16)
    b = oracle.rng_u64(99, 5, 16)
    c = oracle.rng_u64(99, 6, 16)
    assert (a == b).all()
    assert (a != c).any()
    # draw k of a stream = splitmix64(state ^ k * 0x2545f4914f6cdd1d), state from (seed, stream)
    sm = oracle.lib().or_splitmix64
    state = sm(sm(99) ^ ((5 * 0xD1342543DE82EF95) & 0xFFFFFFFFFFFFFFFF))
    for k in range(1, 5):
        assert int(a[k - 1]) == sm(state ^ ((k * 0x2545F4914F6CDD1D) & 0xFFFFFFFFFFFFFFFF))


def test_next_bounded_is_lemire(oracle):
    for bound in (1, 3, 10, 5309, 2**31 + 11):
        v = oracle.rng_bounded(7, 3, bound, 2000)
        assert int(v.max()) < bound
        # restate Lemire on the raw stream: accept iff lo >= 2^32 mod bound
        raw = oracle.rng_u64(7, 3, 6000)
        out, j = [], 0
        while len(out) < 200:
            x = int(raw[j]) >> 32
            j += 1
            m = x * bound
            lo = m & 0xFFFFFFFF
            if lo >= bound or lo >= (2**32) % bound:
                out.append(m >> 32)
        assert out == v[:200].tolist()


def test_sample_quadruple_distinct_and_cache_mapped(oracle):
    # test_registration.cpp:16-33
    cache = np.array([9, 8, 7, 6, 5, 4, 3, 2, 1, 0], np.int32)
    s, t = oracle.sample_quadruples(10, cache, 51, 0, 50)
    for trial in range(50):
        assert len(set(s[trial].tolist())) == 4
        assert ((s[trial] >= 0) & (s[trial] < 10)).all()
        assert (t[trial] == cache[s[trial]]).all()
    a, _ = oracle.sample_quadruples(10, cache, 99, 5, 1)
    b, _ = oracle.sample_quadruples(10, cache, 99, 5, 1)
    assert (a == b).all()


def test_sample_quadruple_errors(oracle):
    import pytest
    cache = np.arange(3, dtype=np.int32)
    with pytest.raises(oracle.OracleError) as e:
        oracle.sample_quadruples(3, cache, 1, 0, 1)
    assert e.value.code == 3  # TooFewPoints
    with pytest.raises(oracle.OracleError) as e:
        oracle.sample_quadruples(10, cache, 1, 0, 1)
    assert e.value.code == 4  # MissingData (cache size mismatch)


def test_prerejected_known_answers(oracle):
    # test_registration.cpp:35-65
    square = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], float)
    assert not oracle.prerejected(square, square, 0.9)
    shrunk = square.copy()
    shrunk[2] = [1, 0.5, 0]
    assert oracle.prerejected(square, shrunk, 0.9)
    rhombus = np.array([[0, 0, 0], [1, 0, 0], [1.5, math.sqrt(3) / 2, 0], [0.5, math.sqrt(3) / 2, 0]])
    for k in range(4):
        assert abs(np.linalg.norm(square[(k + 1) % 4] - square[k]) - np.linalg.norm(rhombus[(k + 1) % 4] - rhombus[k])) < 1e-12
    assert np.linalg.norm(rhombus[2] - rhombus[0]) / np.linalg.norm(square[2] - square[0]) > 1 / 0.9
    assert not oracle.prerejected(square, rhombus, 0.9)
    assert oracle.prerejected(shrunk, square, 0.9)


def test_prerejected_spec_examples(oracle):
    # q edges 0.95 vs p edges 1.0 at tau 0.9 -> accept
    p = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], float)
    assert not oracle.prerejected(p, p * 0.95, 0.9)
    # congruent quadruples are never pre-rejected for tau < 1 (SPEC invariant)
    rng = np.random.default_rng(0)
    for _ in range(50):
        q = rng.normal(size=(4, 3))
        assert not oracle.prerejected(q, q + 0.5, 0.999)
