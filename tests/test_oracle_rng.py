"""Pins for the oracle's random stream: Philox KATs, uniform maps, Box-Muller."""
import math
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _kats():
    rows = []
    for line in open(os.path.join(GOLD, "philox4x32_10_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(x, 16) for x in line.split()]
        rows.append((v[0:4], v[4:6], v[6:10]))
    return rows


def test_philox_known_answers(O):
    for ctr, key, out in _kats():
        assert O.philox4x32_10(ctr, key) == out


def test_word_stream_layout(O):
    # word w of design d is lane w%4 of block q=w/4 at counter (q_lo, q_hi, d, 0), key (seed_lo, seed_hi)
    seed, d = 0x0000002005105494, 77
    for w in [0, 1, 2, 3, 4, 5, 4 * 2**32 + 3, 6 * 10**9 + 1]:
        q = w // 4
        blk = O.philox4x32_10([q & 0xFFFFFFFF, q >> 32, d, 0], [seed & 0xFFFFFFFF, seed >> 32])
        assert O.word(seed, d, w) == blk[w % 4]
    # different designs / seeds give different streams
    a = [O.word(seed, 1, w) for w in range(64)]
    b = [O.word(seed, 2, w) for w in range(64)]
    c = [O.word(seed + 1, 1, w) for w in range(64)]
    assert a != b and a != c


def test_words_per_draw(O):
    # COND: a record of two samples takes p Box-Muller pairs (2p words) + 2 floor(n/2) SOV uniforms,
    # i.e. p + floor(n/2) words per sample; IND: 2*ceil((p+n)/2) words per sample
    assert O.words_per_draw(3, 3, 0) == 4
    assert O.words_per_draw(3, 3, 1) == 6
    assert O.words_per_draw(1, 1, 0) == 1
    assert O.words_per_draw(2, 2, 0) == 3
    assert O.words_per_draw(10, 10, 0) == 15
    assert O.words_per_draw(10, 10, 1) == 20


def _bm(word_r, word_a):
    # u_r = 1 - k 2^-23, u_a = k 2^-23 from the low 23 bits; R = sqrt(-2 ln u_r)
    ur = 1.0 - (word_r & 0x7FFFFF) * 2.0 ** -23
    ua = (word_a & 0x7FFFFF) * 2.0 ** -23
    R = math.sqrt(-2.0 * math.log(ur))
    return R * math.cos(2 * math.pi * ua), R * math.sin(2 * math.pi * ua)


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_cond_record_layout(O, n):
    # COND sample pair (2j, 2j+1) = words [jW, (j+1)W), W = 2n + 2(n/2): sample 2j takes the normals
    # [0, n) of the record's n Box-Muller pairs, sample 2j+1 the normals [n, 2n)
    seed, d = 0x2005105494, 11
    r = [1.0, 0.6, 0.35, 0.2][:n]
    prob = O.point_mass_problem(r, [0.0] * n, 100.0)
    W = 2 * n + 2 * (n // 2)
    for j in [0, 1, 7, 123457]:
        z = []
        for t in range(n):
            z.extend(_bm(O.word(seed, d, j * W + 2 * t), O.word(seed, d, j * W + 2 * t + 1)))
        for h in range(2):
            eps = O.draw(prob, [0.01] * n, O.EST_COND, seed, d, 2 * j + h)["eps"]
            assert np.allclose(eps, z[h * n:(h + 1) * n], rtol=1e-13, atol=1e-13)


def test_cond_pair_halves_independent(O):
    # the two samples of a record share Box-Muller pairs when p is odd (one pair splits across them);
    # the halves must still be independent N(0, I): corr(eps_2j, eps_2j+1) ~ 0, moments of N(0, 1)
    prob = O.point_mass_problem([1, 0.5, 0.25], [0.0, 0.0, 0.0], 100.0)
    eps = np.array([O.draw(prob, [0.01] * 3, O.EST_COND, 99, 5, s)["eps"] for s in range(20000)])
    N = eps.shape[0]
    assert np.all(np.abs(eps.mean(0)) < 5 / math.sqrt(N)) and np.all(np.abs(eps.var(0) - 1) < 5 * math.sqrt(2 / N))
    a, b = eps[0::2], eps[1::2]
    C = np.corrcoef(np.hstack([a, b]).T)
    assert np.all(np.abs(C[np.triu_indices(6, 1)]) < 5 / math.sqrt(N / 2))


def test_word_bits_uniform(O):
    # chi-square on the low 23 bits' top nibble over 40k words: Philox words are uniform
    seed = 12345
    k = np.array([O.word(seed, 3, w) & 0x7FFFFF for w in range(40000)], dtype=np.int64)
    cnt = np.bincount(k >> 19, minlength=16)
    chi2 = ((cnt - 2500.0) ** 2 / 2500.0).sum()
    assert chi2 < 45.0  # chi2_15 99.99th percentile ~ 44.3


def test_box_muller_moments(O):
    # prior normals of the n=3 Formula-10 problem with identity-scaled prior: eps ~ N(0, I)
    prob = O.point_mass_problem([1, 0.5, 0.25], [0.0, 0.0, 0.0], 100.0)
    eps = np.array([O.draw(prob, [0.01, 0.01, 0.01], O.EST_IND, 99, 5, s)["eps"] for s in range(20000)])
    N = eps.shape[0]
    m, v = eps.mean(0), eps.var(0)
    assert np.all(np.abs(m) < 5 / math.sqrt(N))
    assert np.all(np.abs(v - 1) < 5 * math.sqrt(2 / N))
    C = np.corrcoef(eps.T)
    assert np.all(np.abs(C[np.triu_indices(3, 1)]) < 5 / math.sqrt(N))
    # truncation at sqrt(-2 ln 2^-23) = 5.64 (reading R18)
    assert np.abs(eps).max() <= math.sqrt(-2 * math.log(2.0 ** -23)) + 1e-12


def test_null_draws_have_formula1_correlation(O):
    # IND null vector X = L0 W has corr sqrt(r_l/r_k) (Formula 1 / A.1)
    r = [1.0, 0.25]
    prob = O.point_mass_problem(r, [0.0, 0.0], 100.0)
    X = np.array([O.draw(prob, [0.01, 0.01], O.EST_IND, 7, 0, s)["xnull"] for s in range(20000)])
    c = np.corrcoef(X.T)[0, 1]
    assert abs(c - 0.5) < 0.02   # S:137 tolerance, exact sqrt(0.25)
