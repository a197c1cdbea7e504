"""The synthetic-input generators (csrc/host/synth_gen.cpp, host C++ in
libgnna.so; no GPU) against restatements of the reference's draws.

* random_features(n, d, seed) is the reference's function itself
  (pipeline.cpp:57-67): equal to oracle/_ref's ref_random_features, and the
  F32 form is the same doubles rounded.
* The edge samplers draw with std::mt19937_64 and rand.hpp's draw_unit /
  draw_index (rand.hpp:13-21), chunk c of 2^20 pairs from
  mt19937_64(seed + c * 0x9E3779B97F4A7C15): checked against a pure-Python
  mt19937_64 for the first pairs of two chunks, and the output is identical
  across calls (independent of the host's thread scheduling).
"""
import numpy as np
import pytest

MASK64 = (1 << 64) - 1


class MT64:
    """std::mt19937_64 (the 64-bit Mersenne twister of <random>)."""

    def __init__(self, seed):
        self.mt = [0] * 312
        self.mt[0] = seed & MASK64
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & MASK64
        self.i = 312

    def __call__(self):
        if self.i >= 312:
            for k in range(312):
                y = (self.mt[k] & 0xFFFFFFFF80000000) | (self.mt[(k + 1) % 312] & 0x7FFFFFFF)
                v = self.mt[(k + 156) % 312] ^ (y >> 1)
                if y & 1:
                    v ^= 0xB5026F5AA96619E9
                self.mt[k] = v
            self.i = 0
        x = self.mt[self.i]
        self.i += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & MASK64


def draw_unit(rng):
    return (rng() >> 11) * 2.0 ** -53


def draw_index(rng, n):
    return (rng() * n) >> 64


def test_mt64_restatement_matches_std():
    # the standard's check value: the 10000th output of a default-seeded mt19937_64
    rng = MT64(5489)
    for _ in range(9999):
        rng()
    assert rng() == 9981545732273789042


def test_random_features_is_the_references(ref):
    from paper_2006_06608_b200.capi import random_features
    x = random_features(37, 5, 42, np.float64)
    assert np.array_equal(x, ref.random_features(37, 5, 42))
    x32 = random_features(37, 5, 42, np.float32)
    assert np.array_equal(x32, x.astype(np.float32))
    rng = MT64(42)
    assert [draw_unit(rng) for _ in range(5)] == x.reshape(-1)[:5].tolist()


def shuffled_ids(n, seed):
    """planted_partition's Fisher-Yates (pipeline.cpp:37-44) with draw_index."""
    rng = MT64(seed)
    perm = list(range(n))
    for i in range(n, 1, -1):
        j = draw_index(rng, i)
        perm[i - 1], perm[j] = perm[j], perm[i - 1]
    return np.array(perm, np.uint32)


def test_shuffle_is_fisher_yates_relabel():
    from paper_2006_06608_b200.capi import gen_edges
    n, seed = 777, 21
    plain = gen_edges("sbm", n, 3000, seed, shuffle=False, communities=5, p_intra=0.7)
    mixed = gen_edges("sbm", n, 3000, seed, shuffle=True, communities=5, p_intra=0.7)
    perm = shuffled_ids(n, seed ^ 0x9E3779B97F4A7C15)
    assert np.array_equal(mixed, perm[plain])


@pytest.mark.parametrize("shuffle", [False])
def test_sbm_sampler_restated(shuffle):
    from paper_2006_06608_b200.capi import gen_edges
    n, comm, p = 1000, 7, 0.8
    pairs = (1 << 20) + 50  # two chunks
    e = gen_edges("sbm", n, pairs, 9, shuffle=shuffle, communities=comm, p_intra=p)
    assert np.array_equal(e, gen_edges("sbm", n, pairs, 9, shuffle=shuffle, communities=comm, p_intra=p))
    size = n // comm
    for c, first in ((0, 0), (1, 1 << 20)):
        rng = MT64((9 + c * 0x9E3779B97F4A7C15) & MASK64)
        for i in range(first, first + 20):
            src = draw_index(rng, n)
            com = min(src // size, comm - 1)
            base = com * size
            span = n - base if com == comm - 1 else size
            dst = base + draw_index(rng, span) if draw_unit(rng) < p else draw_index(rng, n)
            assert e[i].tolist() == [src, dst], (c, i)


def test_chung_lu_sampler_restated():
    from paper_2006_06608_b200.capi import gen_edges
    n, gamma, i0 = 50000, 2.3, 10.0
    e = gen_edges("chung_lu", n, 4000, 3, gamma=gamma, i0=i0)
    beta = 1.0 / (gamma - 1.0)
    a = 1.0 - beta
    lo, hi = i0 ** a, (n + i0) ** a
    rng = MT64(3)
    for i in range(200):
        for j in range(2):
            x = (lo + draw_unit(rng) * (hi - lo)) ** (1.0 / a) - i0
            f = np.floor(x)
            want = 0 if f <= 0 else (n - 1 if f >= n - 1 else int(f))
            assert abs(int(e[i, j]) - want) <= 1, (i, j)  # pow() may differ in the last ulp across libms
    assert np.array_equal(e, gen_edges("chung_lu", n, 4000, 3, gamma=gamma, i0=i0))
    assert e.max() < n and e.min() >= 0
    # low ids are the hubs
    deg = np.bincount(e.reshape(-1), minlength=n)
    assert deg[:100].sum() > 20 * deg[-100:].sum()
