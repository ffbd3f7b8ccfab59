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


def test_record_sizes(O):
    # records (round 2): COND sample pairs take 2p Box-Muller uniforms + 2 floor(n/2) SOV
    # uniforms, IND sample pairs 2 x 2 ceil((p+n)/2); U uniforms of 23 bits are packed into W = 2 ceil(23 U / 64)
    # words when that is fewer than U (U >= 8), else take one word each
    assert O.record_uniforms(3, 3, 0) == 8 and O.record_words(3, 3, 0) == 6      # 184 bits in 6 words
    assert O.record_uniforms(3, 3, 1) == 12 and O.record_words(3, 3, 1) == 10    # IND: 3 pairs per sample
    assert O.record_uniforms(1, 1, 0) == 2 and O.record_words(1, 1, 0) == 2
    assert O.record_uniforms(2, 2, 0) == 6 and O.record_words(2, 2, 0) == 6
    assert O.record_uniforms(4, 4, 0) == 12 and O.record_words(4, 4, 0) == 10
    assert O.record_uniforms(10, 10, 0) == 30 and O.record_words(10, 10, 0) == 22
    assert O.record_uniforms(10, 10, 1) == 40 and O.record_words(10, 10, 1) == 30
    assert O.record_uniforms(1, 1, 1) == 4 and O.record_words(1, 1, 1) == 4        # 2 ceil(92/64) = 4: unpacked


def _record_bits(O, seed, d, w0, W, tag=0):
    """The record's bit string as one Python integer: bit b is bit (b mod 32) of word w0 + b // 32."""
    return sum(O.word_tagged(seed, d, tag, w0 + j) << (32 * j) for j in range(W))


@pytest.mark.parametrize("U", [2, 6, 8, 12, 30])
def test_record_fields_are_23_bit_slices(O, U):
    # packed records (U >= 8): uniform i = bits [23 i, 23 i + 23) of the little-endian record bit string
    # (big-int slice); unpacked (U <= 6): the low 23 bits of word i
    seed, d = 0x2005105494, 7
    packed = 2 * ((23 * U + 63) // 64) < U
    W = 2 * ((23 * U + 63) // 64) if packed else U
    for w0 in [0, 6 * 1234567, 4 * 2**32 - 2]:
        bits = _record_bits(O, seed, d, w0, W)
        for i in range(U):
            ref = (bits >> (23 * i)) & 0x7FFFFF if packed else O.word_tagged(seed, d, 0, w0 + i) & 0x7FFFFF
            assert O.record_field(seed, d, 0, w0, U, i) == ref, (U, w0, i)


def _bm(kr, ka):
    # u_r = 1 - k 2^-23, u_a = k 2^-23 from 23-bit fields; R = sqrt(-2 ln u_r)
    ur = 1.0 - kr * 2.0 ** -23
    ua = ka * 2.0 ** -23
    R = math.sqrt(-2.0 * math.log(ur))
    return R * math.cos(2 * math.pi * ua), R * math.sin(2 * math.pi * ua)


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_cond_record_layout(O, n):
    # COND sample pair (2j, 2j+1) = record j at words [jW, (j+1)W): sample 2j takes the normals [0, n) of the
    # record's n Box-Muller pairs (fields 2t, 2t+1), sample 2j+1 the normals [n, 2n)
    seed, d = 0x2005105494, 11
    r = [1.0, 0.6, 0.35, 0.2][:n]
    prob = O.point_mass_problem(r, [0.0] * n, 100.0)
    U = 2 * n + 2 * (n // 2)
    packed = 2 * ((23 * U + 63) // 64) < U
    W = 2 * ((23 * U + 63) // 64) if packed else U
    for j in [0, 1, 7, 123457]:
        bits = _record_bits(O, seed, d, j * W, W)
        f = [((bits >> (23 * i)) if packed else (bits >> (32 * i))) & 0x7FFFFF for i in range(U)]
        z = []
        for t in range(n):
            z.extend(_bm(f[2 * t], f[2 * t + 1]))
        for h in range(2):
            eps = O.draw(prob, [0.01] * n, O.EST_COND, seed, d, 2 * j + h)["eps"]
            assert np.allclose(eps, z[h * n:(h + 1) * n], rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("n", [1, 2, 3])
def test_ind_record_layout(O, n):
    # IND sample pair (2j, 2j+1) = record j at words [jW, (j+1)W), U = 4 c uniforms, c = ceil((p+n)/2): sample
    # 2j + h takes Box-Muller pairs [h c, (h+1) c) of the record, its p prior normals first
    seed, d = 0x2005105494, 5
    r = [1.0, 0.6, 0.35][:n]
    prob = O.point_mass_problem(r, [0.0] * n, 100.0)
    c = (2 * n + 1) // 2
    U = 4 * c
    packed = 2 * ((23 * U + 63) // 64) < U
    W = 2 * ((23 * U + 63) // 64) if packed else U
    for j in [0, 3, 98765]:
        bits = _record_bits(O, seed, d, j * W, W)
        f = [((bits >> (23 * i)) if packed else (bits >> (32 * i))) & 0x7FFFFF for i in range(U)]
        for h in range(2):
            z = []
            for t in range(c):
                z.extend(_bm(f[2 * (h * c + t)], f[2 * (h * c + t) + 1]))
            o = O.draw(prob, [0.01] * n, O.EST_IND, seed, d, 2 * j + h)
            assert np.allclose(o["eps"], z[:n], rtol=1e-13, atol=1e-13)
            if n == 1:
                assert np.allclose(o["xnull"], z[n:2 * n], rtol=1e-13, atol=1e-13)


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
